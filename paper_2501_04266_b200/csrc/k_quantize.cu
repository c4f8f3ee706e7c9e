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
#include "quantize_loop.cuh"

namespace hz {
namespace {

using namespace dev;

template <typename T, int B, int BITS, int U, int OUT>
__global__ void __launch_bounds__(kThreads) k_quantize(const T* __restrict__ x, int64_t nblocks,
                                                       uint8_t* __restrict__ codes,
                                                       float* __restrict__ scales,
                                                       const __grid_constant__ SyncArgs sy,
                                                       void* __restrict__ y, int acc) {
  using G = Geo<B>;
  using Emit = typename OutOf<OUT>::E;
  __shared__ __align__(128) float4 stage[OUT >= 3 ? kThreads / 32 : 1][OUT == 4 ? 128 : (OUT >= 3 ? 64 : 1)];
  Emit emit;
  if constexpr (OUT == 1 || OUT == 2) {
    emit.y = static_cast<decltype(emit.y)>(y);
  } else if constexpr (OUT == 3) {
    emit.y = static_cast<float*>(y);
    emit.stage = stage[threadIdx.x >> 5];
    emit.acc = acc;
  } else if constexpr (OUT == 4) {
    emit.y = static_cast<float*>(y);
    emit.stage = stage[threadIdx.x >> 5];
    emit.buf = 0;
  } else if constexpr (OUT == 5 || OUT == 6) {
    emit.y = static_cast<decltype(emit.y)>(y);
    emit.stage = reinterpret_cast<uint4*>(stage[threadIdx.x >> 5]);
    emit.buf = 0;
  }
  if (!sync_wait(sy)) return;   // P2P mode: the readers of what this call overwrites are done
  quantize_loop<T, B, BITS, U, OUT>(x, nblocks, codes, scales, emit, y, acc, global_warp(), num_warps());
  if constexpr (OUT >= 4) emit.finish(threadIdx.x & 31);
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
  // the x_hat stores by TMA: fp32 (HZ_TUNE fb, default on: N = 1 step 3.280 vs 3.301 ms),
  // bf16 / fp16 (HZ_TUNE fbb, default on since the world-1 carveout: round trip 48.5 vs
  // 48.9 us; neutral before it)
  const bool al = (reinterpret_cast<uintptr_t>(y) & 15u) == 0;
  const bool bulk = tune_param("fb", 1) != 0 && al;
  const bool bulk16 = tune_param("fbb", 1) != 0 && al;
  switch (out_dt) {
    case HZ_BF16:
      return bulk16 ? quantize_u<T, 256, BITS, kU, 5>(x, n, codes, scales, st, sy, y, 0)
                    : quantize_u<T, 256, BITS, kU, 1>(x, n, codes, scales, st, sy, y, 0);
    case HZ_F16:
      return bulk16 ? quantize_u<T, 256, BITS, kU, 6>(x, n, codes, scales, st, sy, y, 0)
                    : quantize_u<T, 256, BITS, kU, 2>(x, n, codes, scales, st, sy, y, 0);
    case HZ_F32:
      // no accumulate: the fp32 stores by TMA (HZ_TUNE fb=0: the LSU stores)
      if (!acc && bulk) return quantize_u<T, 256, BITS, kU, 4>(x, n, codes, scales, st, sy, y, 0);
      return quantize_u<T, 256, BITS, kU, 3>(x, n, codes, scales, st, sy, y, acc);
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
                                                               int acc, int order, int chunks, int gbulk,
                                                               const __grid_constant__ SyncArgs sy) {
  // QOUT 3: the quantize job is the round trip of a one-member level (fp32 x_hat into
  // qy, += when acc; codes not stored) — the world-1 backward pair
  __shared__ float4 stage[QOUT == 3 ? kThreads / 32 : 1][QOUT == 3 ? 64 : 1];
  // gbulk: the gathered layer by TMA bulk stores (BulkOut, dequantize_loop.cuh), staged in
  // dynamic shared memory sized by the launcher (0 bytes when off: more L1 for the loads)
  extern __shared__ __align__(128) uint4 gq_gstage[];
  BulkOut bo{gq_gstage + (threadIdx.x >> 5) * (2 * 256 * sizeof(TO) / 16), 0};
  BulkOut* bop = gbulk ? &bo : nullptr;
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
    dequantize_loop<GBITS, TO, GU>(pc, nunits, 8, y, warp, nwarps, 0, INT64_MAX, bop);
  } else {
    dequantize_loop<GBITS, TO, GU>(pc, nunits, 8, y, warp, nwarps, 0, INT64_MAX, bop);
    quantize_loop<T, 256, QBITS, kU, QOUT>(x, nblocks, codes, scales, emit, qy, acc, warp, nwarps);
  }
  if (bop) bulk_out_finish(threadIdx.x & 31);
  sync_signal(sy);
}

template <typename T, int QBITS, int QOUT>
cudaError_t gather_quantize_t(const Pieces& pc, int64_t n_gather, void* y, const void* x, int64_t n_q, uint8_t* codes,
                              float* scales, float* qy, int acc, cudaStream_t st, const SyncArgs& sy) {
  // chunks of the interleaved schedule (HZ_TUNE gqc, default 1 = one pass).  Round 1
  // chose 4 chunks from ~32 gather tiles per warp on (GPT-6.7B / NeoX-20B layers); with
  // the round-2 protocol the one-pass kernel is faster at every size (GPT-6.7B N = 2:
  // 17.96 vs 18.41 ms per step, N = 4: 19.17 vs 19.61; NeoX-20B N = 2: 55.13 vs 55.79,
  // N = 4: 58.12 vs 58.62)
  int chunks = tune_param("gqc", 1);
  if (chunks < 1) chunks = 1;
  // HZ_TUNE gqu=8: 8 gather units in flight per lane (one-pass codes-only variant)
  auto kern = chunks > 1 ? k_gather_quantize<T, QBITS, 8, __nv_bfloat16, QOUT, true>
                         : k_gather_quantize<T, QBITS, 8, __nv_bfloat16, QOUT, false>;
  if constexpr (QOUT == 0)
    if (chunks == 1 && tune_param("gqu", kU) == 8) kern = k_gather_quantize<T, QBITS, 8, __nv_bfloat16, 0, false, 8>;
  const int64_t nunits = n_gather / 8;
  const int64_t nblocks = n_q / 256;
  const int64_t tasks = std::max<int64_t>((nunits + 32 * kU - 1) / (32 * kU), nblocks / (kU * Geo<256>::BPW) + 1);
  // HZ_TUNE gq: 0 = every warp does both jobs, odd CTAs gather first (default); 1 = all
  // gather first; 2 = role split with gqf percent of the CTAs gathering
  int order = tune_param("gq", 0);
  // HZ_TUNE dgb=1: the gathered layer by TMA bulk stores (one-pass schedules only; off by
  // default: N = 2 step 4.06 vs 3.92-3.94 ms, N = 4 4.59 vs 4.43 ms)
  const int gbulk = (order <= 1 && chunks == 1 && tune_param("dgb", 0) != 0 &&
                     (reinterpret_cast<uintptr_t>(y) & 15u) == 0) ? 1 : 0;
  const int dyn = gbulk ? (kThreads / 32) * 2 * 256 * static_cast<int>(sizeof(__nv_bfloat16)) : 0;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), tasks, dyn);
  if (order == 2 && grid < 2) order = 0;
  if (order == 2) {
    int64_t gc = grid * tune_param("gqf", 50) / 100;
    gc = std::min<int64_t>(std::max<int64_t>(gc, 1), grid - 1);
    order = static_cast<int>(2 + gc);
  }
  return launch_k_smem(kern, grid, dyn, st, pc, nunits, static_cast<__nv_bfloat16*>(y), static_cast<const T*>(x),
                       nblocks, codes, scales, qy, acc, order, chunks, gbulk, sy);
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
