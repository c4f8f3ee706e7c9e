// k_quantize (A2 qwZ / A7 qgZ; oracle O4-O5): x (bf16 | fp16 | fp32) ->
// int8 | int4 codes + one fp32 scale per block of B elements.
// Paper: "quantizes blocks of FP16 data into INT8 or INT4 blocks";
// weights INT8 before the all-gather, gradients INT4.
//
// HBM-streaming, no tensor cores.  Mapping: a warp step covers max(B, 256)
// contiguous elements; lane l owns 8 consecutive elements per 256-element
// sub-chunk (one 16-byte bf16 load, one 8/4-byte code store per lane: each warp
// instruction is one contiguous span).  A block's absmax is a shuffle-xor over
// its LPB = min(32, B/8) lanes.  A warp iteration = U full steps (NB = U*BPW
// blocks): all U*NSUB loads are issued first (memory-level parallelism), the
// divisions run once per block (quantize_store), and the main loop has no bounds
// checks so every shuffle is convergent; the last partial iteration (< NB
// blocks) goes through a checked tail path.  Grid-stride over SMs x resident CTAs.
#include "dequantize_loop.cuh"
#include "link.cuh"

namespace hz {
namespace {

using namespace dev;

// OUT: 0 = codes only; 1 / 2 / 3 = also emit the dequantized round trip x_hat as
// bf16 / fp16 / fp32 (+= when acc) — the fused quantize -> dequantize of a level
// whose exchange group has one member (nothing to exchange).
template <int OUT>
struct OutOf;
template <>
struct OutOf<0> { using E = NoEmit; };
template <>
struct OutOf<1> { using E = EmitOut<__nv_bfloat16>; };
template <>
struct OutOf<2> { using E = EmitOut<__half>; };
template <>
struct OutOf<3> { using E = EmitF32; };

// The quantize loop: warp `warp` of `nwarps` processes its grid-stride share of the
// blocks (main loop without bounds checks, then the checked tail on the last warp).
template <typename T, int B, int BITS, int U, int OUT, class Emit>
// Iterations [it0, it1) of the main loop only (U*BPW blocks each; default: all); the
// tail belongs to the range with it1 > the number of full iterations (the last one:
// callers pass INT64_MAX there).
__device__ __forceinline__ void quantize_loop(const T* __restrict__ x, int64_t nblocks, uint8_t* __restrict__ codes,
                                              float* __restrict__ scales, Emit& emit, void* __restrict__ y, int acc,
                                              int64_t warp, int64_t nwarps, int64_t it0 = 0,
                                              int64_t it1 = INT64_MAX) {
  using G = Geo<B>;
  constexpr int NB = U * G::BPW;
  const int lane = threadIdx.x & 31;
  const int lb = lane / G::LPB;
  const int ll = lane % G::LPB;
  const int64_t nfull = nblocks / NB;

  const int64_t itend = it1 < nfull ? it1 : nfull;
  for (int64_t it = it0 + warp; it < itend; it += nwarps) {
    const int64_t blk0 = it * NB;
    In8<T> raw[U][G::NSUB];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t blk = blk0 + u * G::BPW + lb;
#pragma unroll
      for (int k = 0; k < G::NSUB; ++k) raw[u][k].load(x + blk * B + k * G::SUBSTRIDE + ll * 8);
    }
    float v[U][G::NSUB][8];
    float am[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float m = 0.f;
#pragma unroll
      for (int k = 0; k < G::NSUB; ++k) {
        raw[u][k].get(v[u][k]);
#pragma unroll
        for (int i = 0; i < 8; ++i) m = fmaxf(m, fabsf(v[u][k][i]));
      }
      am[u] = group_max<G::LPB>(m);
    }
    quantize_store<B, BITS, U, Emit>(v, am, blk0, lane, codes, scales, emit);
  }

  // tail: the last nblocks % NB blocks, one warp step at a time, bounds-checked
  const int64_t tail0 = nfull * NB;
  if (tail0 < nblocks && warp == nwarps - 1 && it1 > nfull) {
    for (int64_t b0 = tail0; b0 < nblocks; b0 += G::BPW) {
      const int64_t blk = b0 + lb;
      const bool valid = blk < nblocks;
      float v[G::NSUB][8];
      float m = 0.f;
#pragma unroll
      for (int k = 0; k < G::NSUB; ++k) {
        In8<T> r;
        if (valid) {
          r.load(x + blk * B + k * G::SUBSTRIDE + ll * 8);
          r.get(v[k]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) v[k][i] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) m = fmaxf(m, fabsf(v[k][i]));
      }
      m = group_max<G::LPB>(m);
      float scale, inv;
      quant_params<BITS>(m, scale, inv);
#pragma unroll
      for (int k = 0; k < G::NSUB; ++k) {
        unsigned b[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) b[i] = qbits(v[k][i], inv);
        if (valid && codes) {
          Codes8<BITS> out;
          out.set(b);
          out.store(codes + (blk * B + k * G::SUBSTRIDE + ll * 8) * BITS / 8);
        }
        if constexpr (OUT == 1 || OUT == 2) {
          if (valid) {
            float xh[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) xh[i] = __fmul_rn(__fsub_rn(__uint_as_float(b[i]), kMagic), scale);
            emit(blk * B + k * G::SUBSTRIDE + ll * 8, lane, xh);
          }
        } else if constexpr (OUT == 3) {
          // tail (< U blocks): plain per-lane stores, no staging
          float xh[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) xh[i] = __fmul_rn(__fsub_rn(__uint_as_float(b[i]), kMagic), scale);
          if (valid) {
            float* yy = static_cast<float*>(y) + blk * B + k * G::SUBSTRIDE + ll * 8;
#pragma unroll
            for (int i = 0; i < 8; ++i) yy[i] = acc ? __fadd_rn(yy[i], xh[i]) : xh[i];
          }
        }
      }
      if (valid && codes && ll == 0) scales[blk] = scale;
    }
  }
}

template <typename T, int B, int BITS, int U, int OUT>
__global__ void __launch_bounds__(kThreads) k_quantize(const T* __restrict__ x, int64_t nblocks,
                                                       uint8_t* __restrict__ codes,
                                                       float* __restrict__ scales,
                                                       const __grid_constant__ SyncArgs sy,
                                                       void* __restrict__ y, int acc) {
  using G = Geo<B>;
  using Emit = typename OutOf<OUT>::E;
  __shared__ float4 stage[OUT == 3 ? kThreads / 32 : 1][OUT == 3 ? 64 : 1];
  Emit emit;
  if constexpr (OUT == 1 || OUT == 2) {
    emit.y = static_cast<decltype(emit.y)>(y);
  } else if constexpr (OUT == 3) {
    emit.y = static_cast<float*>(y);
    emit.stage = stage[threadIdx.x >> 5];
    emit.acc = acc;
  }
  if (!sync_wait(sy)) return;   // P2P mode: the readers of what this call overwrites are done
  quantize_loop<T, B, BITS, U, OUT>(x, nblocks, codes, scales, emit, y, acc, global_warp(), num_warps());
  sync_signal(sy);   // P2P mode: codes of this phase are ready for the peers
}

constexpr int kU = 4;   // warp steps per warp iteration
// B > 256: NSUB = B/256 loads per step already; B < 256: NB = U*BPW <= 32
constexpr int uq(int B) { return B > 256 ? 1 : kU; }

template <typename T, int B, int BITS, int U, int OUT = 0>
cudaError_t quantize_u(const void* x, int64_t n, uint8_t* codes, float* scales, cudaStream_t st,
                       const SyncArgs& sy, void* y = nullptr, int acc = 0) {
  const int64_t nblocks = n / B;
  constexpr int NB = U * Geo<B>::BPW;
  auto kern = k_quantize<T, B, BITS, U, OUT>;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), nblocks / NB + 1);
  return launch_k(kern, grid, st, static_cast<const T*>(x), nblocks, codes, scales, sy, y, acc);
}

template <typename T, int BITS>
cudaError_t roundtrip_t(const void* x, int64_t n, uint8_t* codes, float* scales, void* y, hz_dtype out_dt,
                        int acc, cudaStream_t st, const SyncArgs& sy) {
  if (tune_param("rt_u", 4) == 2) {   // HZ_TUNE rt_u: 2 (fewer registers, more warps) or 4
    switch (out_dt) {
      case HZ_BF16: return quantize_u<T, 256, BITS, 2, 1>(x, n, codes, scales, st, sy, y, 0);
      case HZ_F16: return quantize_u<T, 256, BITS, 2, 2>(x, n, codes, scales, st, sy, y, 0);
      case HZ_F32: return quantize_u<T, 256, BITS, 2, 3>(x, n, codes, scales, st, sy, y, acc);
    }
    return cudaErrorInvalidValue;
  }
  switch (out_dt) {
    case HZ_BF16: return quantize_u<T, 256, BITS, kU, 1>(x, n, codes, scales, st, sy, y, 0);
    case HZ_F16: return quantize_u<T, 256, BITS, kU, 2>(x, n, codes, scales, st, sy, y, 0);
    case HZ_F32: return quantize_u<T, 256, BITS, kU, 3>(x, n, codes, scales, st, sy, y, acc);
  }
  return cudaErrorInvalidValue;
}

template <typename T, int B, int BITS>
cudaError_t quantize_t(const void* x, int64_t n, uint8_t* codes, float* scales, cudaStream_t st,
                       const SyncArgs& sy) {
  if constexpr (B == 256) {   // HZ_TUNE q_u: 2, 4, 8 (the default block only)
    switch (tune_param("q_u", kU)) {
      case 2: return quantize_u<T, B, BITS, 2>(x, n, codes, scales, st, sy);
      case 8: return quantize_u<T, B, BITS, 8>(x, n, codes, scales, st, sy);
      default: break;
    }
  }
  return quantize_u<T, B, BITS, uq(B)>(x, n, codes, scales, st, sy);
}

template <typename T, int B>
cudaError_t quantize_b(const void* x, int64_t n, int bits, uint8_t* c, float* s, cudaStream_t st,
                       const SyncArgs& sy) {
  return bits == 8 ? quantize_t<T, B, 8>(x, n, c, s, st, sy) : quantize_t<T, B, 4>(x, n, c, s, st, sy);
}

template <typename T>
cudaError_t quantize_d(const void* x, int64_t n, int bits, int block, uint8_t* c, float* s,
                       cudaStream_t st, const SyncArgs& sy) {
  switch (block) {
    case 32: return quantize_b<T, 32>(x, n, bits, c, s, st, sy);
    case 64: return quantize_b<T, 64>(x, n, bits, c, s, st, sy);
    case 128: return quantize_b<T, 128>(x, n, bits, c, s, st, sy);
    case 256: return quantize_b<T, 256>(x, n, bits, c, s, st, sy);
    case 512: return quantize_b<T, 512>(x, n, bits, c, s, st, sy);
    case 1024: return quantize_b<T, 1024>(x, n, bits, c, s, st, sy);
    case 2048: return quantize_b<T, 2048>(x, n, bits, c, s, st, sy);
  }
  return cudaErrorInvalidValue;
}

// k_gather_quantize (P2P transport, B = 256): the gather+dequantize of one phase
// (NVLink-bound: peer code reads) and the quantize of the next phase (HBM-bound),
// two independent jobs, in ONE launch, so that the link and HBM streams overlap
// and one launch / one cross-GPU synchronisation disappears per pair.  Forward:
// gather layer k || quantize layer k+1's primary (the prefetch of
// hz_allgather_params_next); backward: gather layer i-1 || quantize layer i's
// gradient for its reduce-scatter (hz_backward_fused).  Every warp does its
// grid-stride share of both jobs; odd CTAs gather first and even CTAs quantize
// first, so at any time about half the warps stream each resource (HZ_TUNE gq=1:
// every CTA gathers first).  Arithmetic per element is exactly the two kernels'.
template <typename T, int QBITS, int GBITS, typename TO, int QOUT, bool CHUNKED, int GU = kU>
__global__ void __launch_bounds__(kThreads) k_gather_quantize(const __grid_constant__ Pieces pc, int64_t nunits,
                                                               TO* __restrict__ y, const T* __restrict__ x,
                                                               int64_t nblocks, uint8_t* __restrict__ codes,
                                                               float* __restrict__ scales, float* __restrict__ qy,
                                                               int acc, int order, int chunks,
                                                               const __grid_constant__ SyncArgs sy) {
  // QOUT 3: the quantize job is the round trip of a one-member level (fp32 x_hat into
  // qy, += when acc; codes not stored) — the world-1 backward pair
  __shared__ float4 stage[QOUT == 3 ? kThreads / 32 : 1][QOUT == 3 ? 64 : 1];
  using Emit = typename OutOf<QOUT>::E;
  Emit emit;
  if constexpr (QOUT == 3) {
    emit.y = qy;
    emit.stage = stage[threadIdx.x >> 5];
    emit.acc = acc;
  }
  if (!sync_wait(sy)) return;
  const int64_t warp = global_warp(), nwarps = num_warps();
  if (order >= 2) {   // role split: CTAs [0, order - 2) gather only, the rest quantize only
    const int64_t gcta = order - 2;
    const int64_t wpc = kThreads / 32;
    if (blockIdx.x < gcta)
      dequantize_loop<GBITS, TO, GU>(pc, nunits, 8, y, warp, gcta * wpc);
    else
      quantize_loop<T, 256, QBITS, kU, QOUT>(x, nblocks, codes, scales, emit, qy, acc,
                                                     warp - gcta * wpc, nwarps - gcta * wpc);
  } else if (CHUNKED) {
    // both jobs cut into `chunks` consecutive pieces; every warp alternates between
    // them (odd CTAs gather first), so the link and HBM streams stay mixed to the end
    const int64_t ta = (nunits + 32 * GU - 1) / (32 * GU);
    const int64_t tb = nblocks / (kU * Geo<256>::BPW);
    const bool gfirst = blockIdx.x & 1;
    for (int c = 0; c < chunks; ++c) {
      const int64_t a0 = ta * c / chunks, a1 = ta * (c + 1) / chunks;
      const int64_t b0 = tb * c / chunks, b1 = c + 1 == chunks ? INT64_MAX : tb * (c + 1) / chunks;
      if (gfirst) dequantize_loop<GBITS, TO, GU>(pc, nunits, 8, y, warp, nwarps, a0, a1);
      quantize_loop<T, 256, QBITS, kU, QOUT>(x, nblocks, codes, scales, emit, qy, acc, warp, nwarps,
                                                     b0, b1);
      if (!gfirst) dequantize_loop<GBITS, TO, GU>(pc, nunits, 8, y, warp, nwarps, a0, a1);
    }
  } else if (order == 0 && (blockIdx.x & 1) == 0) {
    quantize_loop<T, 256, QBITS, kU, QOUT>(x, nblocks, codes, scales, emit, qy, acc, warp, nwarps);
    dequantize_loop<GBITS, TO, GU>(pc, nunits, 8, y, warp, nwarps);
  } else {
    dequantize_loop<GBITS, TO, GU>(pc, nunits, 8, y, warp, nwarps);
    quantize_loop<T, 256, QBITS, kU, QOUT>(x, nblocks, codes, scales, emit, qy, acc, warp, nwarps);
  }
  sync_signal(sy);
}

// k_gather_quantize_link (P2P transport, B = 256, 8-bit gather, bf16 out, codes-only
// quantize): the dual kernel with the peer pieces moved by TMA bulk copies (link.cuh).
// The work is one atomic queue of CTA-sized tasks: 8192-element tiles of the local
// piece's gather (HBM), 8192-element tiles of the quantize job (HBM) and 16384-element
// tiles of the remote pieces (NVLink), the remote tiles spread evenly through the queue.
//   nlink < 0 (default): every CTA takes any task; a remote tile's bulk copy is issued
//     when the task is taken and consumed (dequantized from shared memory) after the
//     CTA's next HBM task, so the NVLink round trip hides behind HBM work and every SM
//     carries both streams;
//   nlink > 0: CTAs [0, nlink) are dedicated link CTAs streaming the remote tiles
//     through a 3-stage ring, then join the queue of HBM tasks (HZ_TUNE lk=nlink;
//     measured slower: each link CTA is throttled by the HBM CTAs sharing its SM).
// Per-element arithmetic is exactly k_dequantize's and k_quantize's (bitwise parity).
template <typename T, int QBITS>
__global__ void __launch_bounds__(kThreads, 4) k_gather_quantize_link(const __grid_constant__ Pieces pc,
                                                                       __nv_bfloat16* __restrict__ y,
                                                                       const T* __restrict__ x, int64_t nblocks,
                                                                       uint8_t* __restrict__ codes,
                                                                       float* __restrict__ scales, int nlink,
                                                                       LinkGeo lg, const __grid_constant__ SyncArgs sy) {
  extern __shared__ __align__(128) char smem[];
  __shared__ int slot;
  __shared__ int64_t pend[kLinkSMax];
  if (!sync_wait(sy)) return;
  const Ring ring = ring_init(smem, lg.S, lg.stage());
  const LinkTiles lt = link_tiles(pc, lg.te);
  if (nlink > 0 && static_cast<int>(blockIdx.x) < nlink) link_gather<__nv_bfloat16>(pc, lt, y, ring, blockIdx.x, nlink);
  // the local piece (the one piece without its remote bit) as a one-piece gather
  int self = 0;
  while (self < pc.n - 1 && ((pc.remote >> self) & 1u)) ++self;
  Pieces lp{};
  lp.n = 1;
  lp.c[0] = pc.c[self];
  lp.s[0] = pc.s[self];
  lp.len = pc.len;
  const int64_t off = self * pc.len;
  if (pc.sec_c) {
    lp.sec_c = pc.sec_c;
    lp.sec_s = pc.sec_s;
    lp.sec_lo = pc.sec_lo - off;
    lp.sec_hi = pc.sec_hi - off;
  }
  constexpr int GU = kU;                                   // dequantize_loop units per lane
  constexpr int WPC = kThreads / 32;                       // warps per CTA = warp tiles per task
  const int64_t lunits = pc.len / 8;
  const int64_t n_lt = (lunits + 32 * GU * WPC - 1) / (32 * GU * WPC);
  constexpr int NB = kU * Geo<256>::BPW;
  const int64_t nfull = nblocks / NB;
  const int64_t n_qt = (nfull + (nfull * NB < nblocks ? 1 : 0) + WPC - 1) / WPC;
  const int64_t m = n_lt < n_qt ? n_lt : n_qt;
  const int64_t nh = n_lt + n_qt;
  const int64_t nr = nlink > 0 ? 0 : lt.count();           // remote tiles in the queue
  const int64_t total = nh + nr;
  const int64_t wic = threadIdx.x >> 5;
  NoEmit emit;
  int64_t ni = 0, nc = 0;   // remote tiles issued / consumed by this CTA (uniform)
  auto consume_oldest = [&]() {
    mbar_wait(ring.full(nc), ring.parity(nc));
    link_consume<__nv_bfloat16>(pc, lt, pend[nc % lg.S], ring.stage(nc), y);
    ++nc;
    __syncthreads();
  };
  for (;;) {
    const int64_t k = queue_next(sy.queue, &slot);
    if (k >= total) break;
    const int64_t r0 = k * nr / total, r1 = (k + 1) * nr / total;
    if (r1 > r0) {   // remote tile r0: start its copy, consume it after the next HBM task
      if (ni - nc == lg.S) consume_oldest();
      if (threadIdx.x == 0) {
        fence_proxy_async();
        link_issue(pc, lt, r0, ring.stage(ni), ring.full(ni));
        pend[ni % lg.S] = r0;
      }
      ++ni;
      continue;
    }
    const int64_t h = k - r0;   // HBM task h: local gather task a or quantize task b
    int64_t a = -1, b = -1;
    if (h < 2 * m) {
      if (h & 1) b = h >> 1;
      else a = h >> 1;
    } else if (n_lt > n_qt) {
      a = h - m;
    } else {
      b = h - m;
    }
    if (a >= 0) {
      dequantize_loop<8, __nv_bfloat16, GU>(lp, lunits, 8, y + off, wic, WPC, a * WPC, (a + 1) * WPC);
    } else {
      quantize_loop<T, 256, QBITS, kU, 0>(x, nblocks, codes, scales, emit, nullptr, 0, wic, WPC, b * WPC,
                                          b + 1 == n_qt ? INT64_MAX : (b + 1) * WPC);
    }
    if (ni > nc) {
      __syncthreads();   // pend[] written by thread 0 before the HBM task
      consume_oldest();
    }
  }
  while (nc < ni) {
    __syncthreads();
    consume_oldest();
  }
  queue_leave(sy.queue);
  sync_signal(sy);
}

// ring geometry of the link kernels: HZ_TUNE lte (elements per tile, multiple of 1024)
// and ls (stages, 1..kLinkSMax)
LinkGeo link_geo() {
  LinkGeo g{tune_param("lte", 16384), tune_param("ls", 3)};
  g.te = g.te < 1024 ? 1024 : g.te / 1024 * 1024;
  g.S = g.S < 1 ? 1 : (g.S > kLinkSMax ? kLinkSMax : g.S);
  return g;
}

// k_gather_quantize_ws: the same job, warp-specialised instead of queued.  In every
// CTA, warps [0, LW) are link warps: lane 0 of warp 0 streams this CTA's share of the
// remote tiles (tiles b, b + G, ...) through a 3-stage TMA ring and the LW warps
// dequantize each landed tile from shared memory (named barrier 1 among them before a
// stage is re-armed); warps [LW, 8) are HBM warps running the local piece's gather and
// the quantize job grid-stride over all CTAs' HBM warps (odd CTAs gather first, as the
// all-warps kernel).  No CTA-wide barrier after the prologue, no atomics: the HBM warps
// never wait on NVLink latency and the link is fed asynchronously by every SM.
template <typename T, int QBITS, int LW>
__global__ void __launch_bounds__(kThreads, 4) k_gather_quantize_ws(const __grid_constant__ Pieces pc,
                                                                     __nv_bfloat16* __restrict__ y,
                                                                     const T* __restrict__ x, int64_t nblocks,
                                                                     uint8_t* __restrict__ codes,
                                                                     float* __restrict__ scales, LinkGeo lg,
                                                                     const __grid_constant__ SyncArgs sy) {
  extern __shared__ __align__(128) char smem[];
  if (!sync_wait(sy)) return;
  const Ring ring = ring_init(smem, lg.S, lg.stage());
  const int w = threadIdx.x >> 5;
  if (w < LW) {
    const LinkTiles lt = link_tiles(pc, lg.te);
    const int64_t total = lt.count();
    const int64_t mine = total > blockIdx.x ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    if (threadIdx.x == 0) {
      fence_proxy_async();
      for (int64_t i = 0; i < lg.S && i < mine; ++i)
        link_issue(pc, lt, blockIdx.x + i * gridDim.x, ring.stage(i), ring.full(i));
    }
    for (int64_t i = 0; i < mine; ++i) {
      mbar_wait(ring.full(i), ring.parity(i));
      const int64_t t = blockIdx.x + i * gridDim.x;
      int j;
      int64_t e0, cnt;
      link_tile(pc, lt, t, j, e0, cnt);
      const char* stage = ring.stage(i);
      const float* sc = reinterpret_cast<const float*>(stage + lg.te);
      const int64_t g0 = j * pc.len + e0;
      for (int u = threadIdx.x; u < cnt / 8; u += LW * 32) {
        Codes8<8> raw;
        raw.r = *reinterpret_cast<const uint2*>(stage + u * 8);
        const float sv = sc[u >> 5];
        float c[8], v[8];
        raw.decode(c);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __fmul_rn(c[k], sv);
        const int64_t e = g0 + u * 8;
        Out8<__nv_bfloat16>::store(y + e, v);
        if (pc.sec_c && e >= pc.sec_lo && e < pc.sec_hi) {
          raw.store(pc.sec_c + (e - pc.sec_lo));
          if (((e - pc.sec_lo) & 255) == 0) pc.sec_s[(e - pc.sec_lo) >> 8] = sv;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(LW * 32) : "memory");
      if (threadIdx.x == 0 && i + lg.S < mine) {
        fence_proxy_async();
        link_issue(pc, lt, blockIdx.x + (i + lg.S) * gridDim.x, ring.stage(i + lg.S), ring.full(i + lg.S));
      }
    }
  } else {
    int self = 0;
    while (self < pc.n - 1 && ((pc.remote >> self) & 1u)) ++self;
    Pieces lp{};
    lp.n = 1;
    lp.c[0] = pc.c[self];
    lp.s[0] = pc.s[self];
    lp.len = pc.len;
    const int64_t off = self * pc.len;
    if (pc.sec_c) {
      lp.sec_c = pc.sec_c;
      lp.sec_s = pc.sec_s;
      lp.sec_lo = pc.sec_lo - off;
      lp.sec_hi = pc.sec_hi - off;
    }
    constexpr int HW = kThreads / 32 - LW;
    const int64_t hw = static_cast<int64_t>(blockIdx.x) * HW + (w - LW);
    const int64_t nhw = static_cast<int64_t>(gridDim.x) * HW;
    NoEmit emit;
    if (blockIdx.x & 1) {
      dequantize_loop<8, __nv_bfloat16, kU>(lp, pc.len / 8, 8, y + off, hw, nhw);
      quantize_loop<T, 256, QBITS, kU, 0>(x, nblocks, codes, scales, emit, nullptr, 0, hw, nhw);
    } else {
      quantize_loop<T, 256, QBITS, kU, 0>(x, nblocks, codes, scales, emit, nullptr, 0, hw, nhw);
      dequantize_loop<8, __nv_bfloat16, kU>(lp, pc.len / 8, 8, y + off, hw, nhw);
    }
  }
  sync_signal(sy);
}

template <typename T, int QBITS>
cudaError_t gather_quantize_ws_t(const Pieces& pc, void* y, const void* x, int64_t n_q, uint8_t* codes,
                                 float* scales, cudaStream_t st, const SyncArgs& sy) {
  const int lw = tune_param("lw", 2);
  auto kern = lw == 1 ? k_gather_quantize_ws<T, QBITS, 1>
                      : lw == 3 ? k_gather_quantize_ws<T, QBITS, 3> : k_gather_quantize_ws<T, QBITS, 2>;
  const int64_t lunits = pc.len / 8;
  const int64_t tasks = (lunits + 32 * kU - 1) / (32 * kU) + n_q / 256 / kU + 1;
  const LinkGeo lg = link_geo();
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), tasks * 2, lg.smem());
  return launch_k_smem(kern, grid, lg.smem(), st, pc, static_cast<__nv_bfloat16*>(y), static_cast<const T*>(x),
                       n_q / 256, codes, scales, lg, sy);
}

template <typename T, int QBITS>
cudaError_t gather_quantize_link_t(const Pieces& pc, void* y, const void* x, int64_t n_q, uint8_t* codes,
                                   float* scales, int nlink, cudaStream_t st, const SyncArgs& sy) {
  auto kern = k_gather_quantize_link<T, QBITS>;
  const int64_t lunits = pc.len / 8;
  const LinkGeo lg = link_geo();
  const int64_t remote_tiles = int64_t(pc.n - 1) * ((pc.len + lg.te - 1) / lg.te);
  const int64_t tasks = (lunits + 32 * kU - 1) / (32 * kU) + n_q / 256 / kU + 1 + remote_tiles * 8;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), tasks, lg.smem());
  if (nlink > 0 && grid <= nlink) nlink = static_cast<int>(std::max<int64_t>(1, grid / 2));
  return launch_k_smem(kern, grid, lg.smem(), st, pc, static_cast<__nv_bfloat16*>(y), static_cast<const T*>(x),
                       n_q / 256, codes, scales, nlink, lg, sy);
}

// link CTAs of the role-split kernels (HZ_TUNE lk: 0 = the all-warps schedule)
int link_ctas(const Pieces& pc, const SyncArgs& sy) {
  if (!sy.queue || !pc.remote || pc.n < 2) return 0;
  int nrem = 0;
  for (int j = 0; j < pc.n; ++j) nrem += (pc.remote >> j) & 1u;
  if (nrem != pc.n - 1 || (pc.len % 1024) != 0) return 0;
  // -2: warp-specialised (default); -1: every CTA through the queue; > 0: dedicated link
  // CTAs; 0: off (the all-warps kernels with per-lane peer loads)
  const int lk = tune_param("lk", -2);
  if (lk == 0) return 0;
  if (lk < 0) return lk < -1 ? -2 : -1;
  const int64_t tiles = int64_t(nrem) * ((pc.len + link_geo().te - 1) / link_geo().te);
  return static_cast<int>(std::min<int64_t>(lk, tiles));
}

template <typename T, int QBITS, int QOUT>
cudaError_t gather_quantize_t(const Pieces& pc, int64_t n_gather, void* y, const void* x, int64_t n_q, uint8_t* codes,
                              float* scales, float* qy, int acc, cudaStream_t st, const SyncArgs& sy) {
  if constexpr (QOUT == 0) {
    const int nlink = link_ctas(pc, sy);
    if (nlink == -2) return gather_quantize_ws_t<T, QBITS>(pc, y, x, n_q, codes, scales, st, sy);
    if (nlink != 0) return gather_quantize_link_t<T, QBITS>(pc, y, x, n_q, codes, scales, nlink, st, sy);
  }
  // chunks of the interleaved schedule (HZ_TUNE gqc; default by size): one pass when a
  // warp has few gather tiles (GPT-1.3B layer, ~10 per warp: the chunked kernel's extra
  // registers cost more than the balance gains, 3.80 vs 4.20 ms), 4 chunks from ~32 tiles
  // per warp on (GPT-6.7B layer: 19.28 -> 17.76 ms per step at N = 2)
  int chunks = tune_param("gqc", 0);
  if (chunks <= 0) {
    const int64_t per_warp = (n_gather / 8 + 32 * kU - 1) / (32 * kU) / (int64_t(sm_count()) * 32);
    chunks = per_warp >= 32 ? 4 : 1;
  }
  // HZ_TUNE gqu=8: 8 gather units in flight per lane (one-pass codes-only variant)
  auto kern = chunks > 1 ? k_gather_quantize<T, QBITS, 8, __nv_bfloat16, QOUT, true>
                         : k_gather_quantize<T, QBITS, 8, __nv_bfloat16, QOUT, false>;
  if constexpr (QOUT == 0)
    if (chunks == 1 && tune_param("gqu", kU) == 8) kern = k_gather_quantize<T, QBITS, 8, __nv_bfloat16, 0, false, 8>;
  const int64_t nunits = n_gather / 8;
  const int64_t nblocks = n_q / 256;
  const int64_t tasks = std::max<int64_t>((nunits + 32 * kU - 1) / (32 * kU), nblocks / (kU * Geo<256>::BPW) + 1);
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), tasks);
  // HZ_TUNE gq: 0 = every warp does both jobs, odd CTAs gather first (default); 1 = all
  // gather first; 2 = role split with gqf percent of the CTAs gathering
  int order = tune_param("gq", 0);
  if (order == 2 && grid < 2) order = 0;
  if (order == 2) {
    int64_t gc = grid * tune_param("gqf", 50) / 100;
    gc = std::min<int64_t>(std::max<int64_t>(gc, 1), grid - 1);
    order = static_cast<int>(2 + gc);
  }
  // HZ_TUNE gqc: chunks of the interleaved schedule (order 0)
  return launch_k(kern, grid, st, pc, nunits, static_cast<__nv_bfloat16*>(y), static_cast<const T*>(x), nblocks,
                  codes, scales, qy, acc, order, chunks, sy);
}

template <typename T>
cudaError_t gather_quantize_d(const Pieces& pc, int64_t n_gather, void* y, const void* x, int64_t n_q, int qbits,
                              uint8_t* codes, float* scales, float* qy, int acc, cudaStream_t st, const SyncArgs& sy) {
  if (qy)
    return qbits == 8 ? gather_quantize_t<T, 8, 3>(pc, n_gather, y, x, n_q, codes, scales, qy, acc, st, sy)
                      : gather_quantize_t<T, 4, 3>(pc, n_gather, y, x, n_q, codes, scales, qy, acc, st, sy);
  return qbits == 8 ? gather_quantize_t<T, 8, 0>(pc, n_gather, y, x, n_q, codes, scales, nullptr, 0, st, sy)
                    : gather_quantize_t<T, 4, 0>(pc, n_gather, y, x, n_q, codes, scales, nullptr, 0, st, sy);
}

}  // namespace

bool roundtrip_supported(int block) { return block == 256; }

cudaError_t launch_quantize_roundtrip(const void* x, hz_dtype dt, int64_t n, int bits, int block,
                                      uint8_t* codes, float* scales, void* y, hz_dtype out_dt, int acc,
                                      cudaStream_t st, const SyncArgs* sync) {
  const SyncArgs sy = sync ? *sync : SyncArgs{};
  if (block != 256) return cudaErrorInvalidValue;
  if (n == 0 && !sync) return cudaSuccess;
  {
    const cudaError_t e = tiles_quantize(x, dt, n, bits, block, codes, scales, y, out_dt, acc, st, sy);
    if (e != cudaErrorNotSupported) return e;
  }
  switch (dt) {
    case HZ_F32:
      return bits == 8 ? roundtrip_t<float, 8>(x, n, codes, scales, y, out_dt, acc, st, sy)
                       : roundtrip_t<float, 4>(x, n, codes, scales, y, out_dt, acc, st, sy);
    case HZ_BF16:
      return bits == 8 ? roundtrip_t<__nv_bfloat16, 8>(x, n, codes, scales, y, out_dt, acc, st, sy)
                       : roundtrip_t<__nv_bfloat16, 4>(x, n, codes, scales, y, out_dt, acc, st, sy);
    case HZ_F16:
      return bits == 8 ? roundtrip_t<__half, 8>(x, n, codes, scales, y, out_dt, acc, st, sy)
                       : roundtrip_t<__half, 4>(x, n, codes, scales, y, out_dt, acc, st, sy);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_quantize(const void* x, hz_dtype dt, int64_t n, int bits, int block,
                            uint8_t* codes, float* scales, cudaStream_t st, const SyncArgs* sync) {
  const SyncArgs sy = sync ? *sync : SyncArgs{};
  if (n == 0 && !sync) return cudaSuccess;
  {
    const cudaError_t e = tiles_quantize(x, dt, n, bits, block, codes, scales, nullptr, HZ_BF16, 0, st, sy);
    if (e != cudaErrorNotSupported) return e;
  }
  switch (dt) {
    case HZ_F32: return quantize_d<float>(x, n, bits, block, codes, scales, st, sy);
    case HZ_BF16: return quantize_d<__nv_bfloat16>(x, n, bits, block, codes, scales, st, sy);
    case HZ_F16: return quantize_d<__half>(x, n, bits, block, codes, scales, st, sy);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hz

namespace hz {

// The standalone gather+dequantize (k_dequantize's job) through the link-CTA kernel:
// no quantize tasks in the queue.  cudaErrorNotSupported when the pieces do not qualify
// (no remote piece, not a P2P launch, HZ_TUNE lk=0).
cudaError_t launch_gather_link(const Pieces& pc, void* y, cudaStream_t st, const SyncArgs& sy) {
  const int nlink = link_ctas(pc, sy);
  if (nlink == 0) return cudaErrorNotSupported;
  if (nlink == -2) return gather_quantize_ws_t<__nv_bfloat16, 8>(pc, y, nullptr, 0, nullptr, nullptr, st, sy);
  return gather_quantize_link_t<__nv_bfloat16, 8>(pc, y, nullptr, 0, nullptr, nullptr, nlink, st, sy);
}

bool gather_quantize_supported(int block, int gather_bits, hz_dtype out_dt) {
  return block == 256 && gather_bits == 8 && out_dt == HZ_BF16;
}

cudaError_t launch_gather_quantize(const Pieces& pc, int64_t n_gather, void* y, const void* x, hz_dtype dt,
                                   int64_t n_q, int qbits, uint8_t* codes, float* scales, float* qy, int acc,
                                   cudaStream_t st, const SyncArgs& sy) {
  if (pc.n * pc.len == n_gather) {
    const cudaError_t e = tiles_dual(pc, y, x, dt, n_q, qbits, codes, scales, qy, acc, st, sy);
    if (e != cudaErrorNotSupported) return e;
  }
  switch (dt) {
    case HZ_F32: return gather_quantize_d<float>(pc, n_gather, y, x, n_q, qbits, codes, scales, qy, acc, st, sy);
    case HZ_BF16:
      return gather_quantize_d<__nv_bfloat16>(pc, n_gather, y, x, n_q, qbits, codes, scales, qy, acc, st, sy);
    case HZ_F16: return gather_quantize_d<__half>(pc, n_gather, y, x, n_q, qbits, codes, scales, qy, acc, st, sy);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hz
