// Level reduce of the qgZ reduce-scatter (A9 / A10; oracle O9 `reduce_coded`):
// g coded chunks (the members of one level exchange group, ascending level
// digit) -> x_hat_p = fl(code*scale) -> acc = ((x_hat_0 + x_hat_1) + ...) in
// fp32, one rounding per add (R10), then
//   k_reduce_requant: requantize acc (int4 | int8) into the next level's send
//                     layout (same SoA arrays, this chunk's range) — the fused
//                     dequant+sum+requant that keeps the all-to-all design free
//                     of repeated error accumulation within a level;
//   k_reduce_f32:     write the fp32 gradient shard, or add it to the shard
//                     (A = fl(A + acc), gradient accumulation).
//
// k_reduce_requant needs a block-wide absmax, so it uses the block-grouped
// mapping of k_quantize.  k_reduce_f32 has no cross-element step, so it uses an
// elementwise mapping with one 8-byte code load per lane per input and a
// shared-memory transpose for coalesced 512-byte fp32 stores.  Inputs may be
// peer-mapped (NVLink P2P transport): 8-byte loads keep peer reads at full speed.
#include "dequantize_loop.cuh"
#include "quantize_loop.cuh"
#include "reduce_loop.cuh"

namespace hz {
namespace {

using namespace dev;


// ------------------------------------------------------------ requantizing reduce
// Sum of the inputs for U warp steps starting at block blk0 (this lane's 8-element
// sub-chunks).  GT > 0: exactly GT inputs, every load of the U steps issued before
// any sum.  GT == 0: runtime a.g inputs, one input at a time.  `valid` masks
// steps past the end (tail path only; the main loop passes all-true).
template <int B, int BIN, int GT, int U>
__device__ __forceinline__ void sum_steps(const RedArgs& a, int64_t blk0, int lane, const bool (&valid)[U],
                                          float (&acc)[U][Geo<B>::NSUB][8]) {
  using G = Geo<B>;
  const int lb = lane / G::LPB;
  const int ll = lane % G::LPB;
  if constexpr (GT > 0) {
    Codes8<BIN> raw[U][GT][G::NSUB];
    float sc[U][GT];
    if constexpr (B == 256 && U == 4) {
      // main loop only (the tail uses U = 1): blk0 % 4 == 0, all steps valid; the
      // 4 scales of an input are one 16-byte broadcast load
#pragma unroll
      for (int p = 0; p < GT; ++p) {
        const float4 s4 = HZ_PEER_LD(reinterpret_cast<const float4*>(a.s[p] + blk0));
        sc[0][p] = s4.x;
        sc[1][p] = s4.y;
        sc[2][p] = s4.z;
        sc[3][p] = s4.w;
#pragma unroll
        for (int u = 0; u < U; ++u) raw[u][p][0].load(a.c[p] + ((blk0 + u) * B + ll * 8) * BIN / 8);
      }
    } else {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t blk = blk0 + u * G::BPW + lb;
#pragma unroll
      for (int p = 0; p < GT; ++p) {
        sc[u][p] = 0.f;
        if (valid[u]) {
#pragma unroll
          for (int k = 0; k < G::NSUB; ++k)
            raw[u][p][k].load(a.c[p] + (blk * B + k * G::SUBSTRIDE + ll * 8) * BIN / 8);
          sc[u][p] = HZ_PEER_LD(a.s[p] + blk);
        } else {
#pragma unroll
          for (int k = 0; k < G::NSUB; ++k) raw[u][p][k].zero();
        }
      }
    }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int k = 0; k < G::NSUB; ++k) {
        float c[8];
        raw[u][0][k].decode(c);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[u][k][i] = __fmul_rn(c[i], sc[u][0]);
#pragma unroll
        for (int p = 1; p < GT; ++p) {
          raw[u][p][k].decode(c);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[u][k][i] = __fadd_rn(acc[u][k][i], __fmul_rn(c[i], sc[u][p]));
        }
      }
    }
  } else {
    for (int p = 0; p < a.g; ++p) {
      Codes8<BIN> raw[U][G::NSUB];
      float sc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t blk = blk0 + u * G::BPW + lb;
        sc[u] = 0.f;
        if (valid[u]) {
#pragma unroll
          for (int k = 0; k < G::NSUB; ++k)
            raw[u][k].load(a.c[p] + (blk * B + k * G::SUBSTRIDE + ll * 8) * BIN / 8);
          sc[u] = HZ_PEER_LD(a.s[p] + blk);
        } else {
#pragma unroll
          for (int k = 0; k < G::NSUB; ++k) raw[u][k].zero();
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < G::NSUB; ++k) {
          float c[8];
          raw[u][k].decode(c);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float xh = __fmul_rn(c[i], sc[u]);
            acc[u][k][i] = p == 0 ? xh : __fadd_rn(acc[u][k][i], xh);
          }
        }
    }
  }
}

// Main loop: warp iterations of U full steps (NB = U*BPW blocks), no bounds checks,
// quantize_store epilogue (one division per block).  Tail (< NB blocks): one
// checked step at a time by the last warp.
template <int B, int BIN, int BOUT, int GT, int U>
__global__ void __launch_bounds__(kThreads) k_reduce_requant(const __grid_constant__ RedArgs a,
                                                             const __grid_constant__ SyncArgs sy) {
  using G = Geo<B>;
  if (!sync_wait(sy)) return;   // P2P: peers' chunks ready, and nobody still reads our output slot
  constexpr int NB = U * G::BPW;
  const int lane = threadIdx.x & 31;
  const int lb = lane / G::LPB;
  const int ll = lane % G::LPB;
  const int64_t warp = global_warp();
  const int64_t nwarps = num_warps();
  const int64_t nblocks = a.n / B;
  const int64_t nfull = nblocks / NB;

  for (int64_t it = warp; it < nfull; it += nwarps) {
    const int64_t blk0 = it * NB;
    bool valid[U];
#pragma unroll
    for (int u = 0; u < U; ++u) valid[u] = true;
    float acc[U][G::NSUB][8];
    sum_steps<B, BIN, GT, U>(a, blk0, lane, valid, acc);
    float am[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float m = 0.f;
#pragma unroll
      for (int k = 0; k < G::NSUB; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) m = fmaxf(m, fabsf(acc[u][k][i]));
      am[u] = group_max<G::LPB>(m);
    }
    quantize_store<B, BOUT, U, NoEmit>(acc, am, blk0, lane, a.oc, a.os, NoEmit{});
  }

  const int64_t tail0 = nfull * NB;
  if (tail0 < nblocks && warp == nwarps - 1) {
    for (int64_t b0 = tail0; b0 < nblocks; b0 += G::BPW) {
      const int64_t blk = b0 + lb;
      bool valid[1] = {blk < nblocks};
      float acc[1][G::NSUB][8];
      sum_steps<B, BIN, GT, 1>(a, b0, lane, valid, acc);
      float m = 0.f;
#pragma unroll
      for (int k = 0; k < G::NSUB; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) m = fmaxf(m, valid[0] ? fabsf(acc[0][k][i]) : 0.f);
      m = group_max<G::LPB>(m);
      float scale, inv;
      quant_params<BOUT>(m, scale, inv);
      if (valid[0]) {
#pragma unroll
        for (int k = 0; k < G::NSUB; ++k) {
          unsigned bq[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) bq[i] = qbits(acc[0][k][i], inv);
          Codes8<BOUT> out;
          out.set(bq);
          out.store(a.oc + (blk * B + k * G::SUBSTRIDE + ll * 8) * BOUT / 8);
        }
        if (ll == 0) a.os[blk] = scale;
      }
    }
  }
  sync_signal(sy);   // P2P: done reading this level, next level's chunks ready
}

// --------------------------------------------------------------- fp32-output reduce
// Elementwise: a unit is the 8 code bytes of E = 64/BIN consecutive elements (one
// 8-byte load per input — wide enough for NVLink peer reads, which run at half
// speed with 2-byte loads); a warp chunk is 32 consecutive units.  The E fp32 sums
// of a lane are staged through shared memory (XOR-swizzled 16-byte granules:
// conflict-free both ways) so that every global store / accumulate load of the
// warp is one contiguous 512-byte span.
template <int BIN>
struct Wide;
template <>
struct Wide<8> {
  static constexpr int E = 8;
  uint2 r;
  __device__ __forceinline__ void load(const uint8_t* p) { r = HZ_PEER_LD(reinterpret_cast<const uint2*>(p)); }
  __device__ __forceinline__ void decode(float (&c)[E]) const {
    Codes8<8> x;
    x.r = r;
    x.decode(c);
  }
};
template <>
struct Wide<4> {
  static constexpr int E = 16;
  uint2 r;
  __device__ __forceinline__ void load(const uint8_t* p) { r = HZ_PEER_LD(reinterpret_cast<const uint2*>(p)); }
  __device__ __forceinline__ void decode(float (&c)[E]) const {
    Codes8<4> lo, hi;
    lo.r = r.x;
    hi.r = r.y;
    float a[8], b[8];
    lo.decode(a);
    hi.decode(b);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      c[i] = a[i];
      c[8 + i] = b[i];
    }
  }
};

template <int BIN, int GT, int U, bool ACC>
__global__ void __launch_bounds__(kThreads) k_reduce_f32(const __grid_constant__ RedArgs a, int log2b,
                                                         const __grid_constant__ SyncArgs sy) {
  __shared__ float4 stage[kThreads / 32][32 * red_granules<BIN>()];
  if (!sync_wait(sy)) return;
  reduce_f32_loop<BIN, GT, U, ACC>(a, log2b, stage[threadIdx.x >> 5], global_warp(), num_warps());
  sync_signal(sy);
}

// ---------------------------------------------------------------------- launch
constexpr int kUR = 4;   // warp steps per warp iteration (requant)
constexpr int kUF = 2;   // 8-byte code units in flight per lane per input (fp32 out)
constexpr int ur(int B) { return B > 256 ? 1 : kUR; }

template <int B, int BIN, int BOUT, int GT, int U>
cudaError_t requant_u(const RedArgs& a, cudaStream_t st, const SyncArgs& sy) {
  constexpr int NB = U * Geo<B>::BPW;
  auto kern = k_reduce_requant<B, BIN, BOUT, GT, U>;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), a.n / B / NB + 1);
  return launch_k(kern, grid, st, a, sy);
}

template <int B, int BIN, int BOUT, int GT>
cudaError_t requant_t(const RedArgs& a, cudaStream_t st, const SyncArgs& sy) {
  if constexpr (B == 256 && GT > 0 && GT <= 2) {   // HZ_TUNE rq_u: 1, 2, 4
    switch (tune_param("rq_u", kUR)) {
      case 1: return requant_u<B, BIN, BOUT, GT, 1>(a, st, sy);
      case 2: return requant_u<B, BIN, BOUT, GT, 2>(a, st, sy);
      default: break;
    }
  }
  return requant_u<B, BIN, BOUT, GT, ur(B)>(a, st, sy);
}

template <int B, int BIN, int BOUT>
cudaError_t requant_g(const RedArgs& a, cudaStream_t st, const SyncArgs& sy) {
  // Unrolled input prefetch for the common group sizes; large blocks with many
  // inputs use the one-input-at-a-time loop (register budget).
  switch (a.g) {
    case 1: return requant_t<B, BIN, BOUT, 1>(a, st, sy);
    case 2: return requant_t<B, BIN, BOUT, 2>(a, st, sy);
    case 4: return B >= 1024 ? requant_t<B, BIN, BOUT, 0>(a, st, sy) : requant_t<B, BIN, BOUT, 4>(a, st, sy);
    case 8: return B >= 512 ? requant_t<B, BIN, BOUT, 0>(a, st, sy) : requant_t<B, BIN, BOUT, 8>(a, st, sy);
    default: return requant_t<B, BIN, BOUT, 0>(a, st, sy);
  }
}

template <int B>
cudaError_t requant_b(const RedArgs& a, int bits_in, int bits_out, cudaStream_t st, const SyncArgs& sy) {
  if (bits_in == 8) return bits_out == 8 ? requant_g<B, 8, 8>(a, st, sy) : requant_g<B, 8, 4>(a, st, sy);
  return bits_out == 8 ? requant_g<B, 4, 8>(a, st, sy) : requant_g<B, 4, 4>(a, st, sy);
}

template <int BIN, int GT, int U>
cudaError_t f32_u(const RedArgs& a, int log2b, cudaStream_t st, const SyncArgs& sy) {
  const int64_t nunits = a.n / Wide<BIN>::E;
  auto kern = a.accumulate ? k_reduce_f32<BIN, GT, U, true> : k_reduce_f32<BIN, GT, U, false>;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), (nunits + 32 * U - 1) / (32 * U));
  return launch_k(kern, grid, st, a, log2b, sy);
}

template <int BIN, int GT>
cudaError_t f32_t(const RedArgs& a, int log2b, cudaStream_t st, const SyncArgs& sy) {
  if constexpr (GT > 0 && GT <= 2) {   // HZ_TUNE rf_u: 1, 2, 4
    switch (tune_param("rf_u", kUF)) {
      case 1: return f32_u<BIN, GT, 1>(a, log2b, st, sy);
      case 4: return f32_u<BIN, GT, 4>(a, log2b, st, sy);
      default: break;
    }
  }
  return f32_u<BIN, GT, kUF>(a, log2b, st, sy);
}

template <int BIN>
cudaError_t f32_g(const RedArgs& a, int log2b, cudaStream_t st, const SyncArgs& sy) {
  switch (a.g) {
    case 1: return f32_t<BIN, 1>(a, log2b, st, sy);
    case 2: return f32_t<BIN, 2>(a, log2b, st, sy);
    case 4: return f32_t<BIN, 4>(a, log2b, st, sy);
    case 8: return f32_t<BIN, 8>(a, log2b, st, sy);
    default: return f32_t<BIN, 0>(a, log2b, st, sy);
  }
}

constexpr int kUF_ = 2;   // = kUF: 8-byte code units in flight per lane per input (fp32 out)

// ------------------------------------------------------------ backward triple kernel
// k_gather_quantize_reduce (P2P transport, the backward step of layer i-1 with the
// deferred last qgZ hop of layer i): three independent jobs of three phases in ONE
// launch — the hpZ gather+dequantize of layer i-2 (NVLink + HBM writes), the int4 / int8
// quantize of layer i-1's gradient into its send buffer (HBM reads) and the fp32 level
// reduce of layer i (NVLink + HBM writes) — so the HBM-read and the link/write-heavy
// streams overlap and one launch, one cross-GPU wait and one publication disappear per
// layer.  Every warp does its grid-stride share of all three; CTAs rotate the order
// (blockIdx % 3) so that each job is being streamed by a third of the GPU at any time.
// Per-element arithmetic is exactly k_dequantize's, k_quantize's and k_reduce_f32's.
// each job a separate (non-inlined) function: one register allocation each, so the
// kernel keeps 4 CTAs per SM (64 registers) instead of the union of the three loops'
template <typename T, int QBITS>
__device__ __noinline__ void gqr_quantize(const T* __restrict__ x, int64_t nblocks, uint8_t* __restrict__ codes,
                                          float* __restrict__ scales, int64_t warp, int64_t nwarps) {
  NoEmit emit;
  quantize_loop<T, 256, QBITS, 4, 0>(x, nblocks, codes, scales, emit, nullptr, 0, warp, nwarps);
}
__device__ __noinline__ void gqr_gather(const Pieces& pc, int64_t nunits, __nv_bfloat16* __restrict__ y,
                                        int64_t warp, int64_t nwarps, BulkOut* bo) {
  dequantize_loop<8, __nv_bfloat16, 4>(pc, nunits, 8, y, warp, nwarps, 0, INT64_MAX, bo);
}
template <int RBIN, int RGT, bool RACC>
__device__ __noinline__ void gqr_reduce(const RedArgs& ra, int log2b, float4* st, int64_t warp, int64_t nwarps) {
  reduce_f32_loop<RBIN, RGT, 2, RACC>(ra, log2b, st, warp, nwarps);
}

template <typename T, int QBITS, int RBIN, int RGT, bool RACC>
__global__ void __launch_bounds__(kThreads, 4) k_gather_quantize_reduce(
    const __grid_constant__ Pieces pc, int64_t nunits, __nv_bfloat16* __restrict__ y, const T* __restrict__ x,
    int64_t nblocks, uint8_t* __restrict__ codes, float* __restrict__ scales, const __grid_constant__ RedArgs ra,
    int log2b, int gbulk, int jorder, const __grid_constant__ SyncArgs sy) {
  __shared__ float4 stage[kThreads / 32][32 * red_granules<RBIN>()];
  // gbulk: the bulk-store staging of the gathered layer, in dynamic shared memory sized by
  // the launcher (0 bytes when off: a smaller shared-memory configuration leaves more L1
  // for the loads in flight)
  extern __shared__ __align__(128) uint4 gqr_gstage[];
  if (!sync_wait(sy)) return;
  const int64_t warp = global_warp(), nwarps = num_warps();
  float4* st = stage[threadIdx.x >> 5];
  BulkOut bo{gqr_gstage + (threadIdx.x >> 5) * (2 * 256 * 2 / 16), 0};
  BulkOut* bop = gbulk ? &bo : nullptr;
  // job order per CTA (HZ_TUNE gqro): 0 = rotate by blockIdx % 3 (default); 1 = quantize,
  // gather, reduce; 2 = gather, reduce, quantize; 3 = even CTAs quantize first, odd CTAs
  // gather first, reduce last
  int seq[3];
  if (jorder == 1) {
    seq[0] = 1; seq[1] = 0; seq[2] = 2;
  } else if (jorder == 2) {
    seq[0] = 0; seq[1] = 2; seq[2] = 1;
  } else if (jorder == 3) {
    seq[0] = (blockIdx.x & 1) ? 0 : 1; seq[1] = (blockIdx.x & 1) ? 1 : 0; seq[2] = 2;
  } else {
    const int o = static_cast<int>(blockIdx.x % 3);
    seq[0] = o; seq[1] = (o + 1) % 3; seq[2] = (o + 2) % 3;
  }
#pragma unroll 1
  for (int k = 0; k < 3; ++k) {
    const int job = seq[k];
    if (job == 0) gqr_gather(pc, nunits, y, warp, nwarps, bop);
    else if (job == 1) gqr_quantize<T, QBITS>(x, nblocks, codes, scales, warp, nwarps);
    else gqr_reduce<RBIN, RGT, RACC>(ra, log2b, st, warp, nwarps);
  }
  if (bop) bulk_out_finish(threadIdx.x & 31);
  sync_signal(sy);
}

template <typename T, int QBITS, int RBIN, int RGT, bool RACC>
cudaError_t gqr_t(const Pieces& pc, int64_t n_gather, void* y, const void* x, int64_t n_q, uint8_t* codes,
                  float* scales, const RedArgs& ra, cudaStream_t st, const SyncArgs& sy) {
  auto kern = k_gather_quantize_reduce<T, QBITS, RBIN, RGT, RACC>;
  constexpr int E = Wide<RBIN>::E;
  const int64_t tasks = std::max<int64_t>(std::max<int64_t>(n_gather / 8 / (32 * 4), n_q / 256 / 4),
                                          ra.n / E / (32 * kUF_)) + 1;
  const int gbulk = tune_param("dgb", 0) != 0 && (reinterpret_cast<uintptr_t>(y) & 15u) == 0 ? 1 : 0;
  const int dyn = gbulk ? (kThreads / 32) * 2 * 256 * 2 : 0;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), tasks, dyn);
  return launch_k_smem(kern, grid, dyn, st, pc, n_gather / 8, static_cast<__nv_bfloat16*>(y),
                       static_cast<const T*>(x), n_q / 256, codes, scales, ra, 8, gbulk, tune_param("gqro", 0), sy);
}

template <typename T, int QBITS, int RBIN>
cudaError_t gqr_g(const Pieces& pc, int64_t n_gather, void* y, const void* x, int64_t n_q, uint8_t* codes,
                  float* scales, const RedArgs& ra, cudaStream_t st, const SyncArgs& sy) {
  switch (ra.g) {
    case 2: return ra.accumulate ? gqr_t<T, QBITS, RBIN, 2, true>(pc, n_gather, y, x, n_q, codes, scales, ra, st, sy)
                                 : gqr_t<T, QBITS, RBIN, 2, false>(pc, n_gather, y, x, n_q, codes, scales, ra, st, sy);
    case 4: return ra.accumulate ? gqr_t<T, QBITS, RBIN, 4, true>(pc, n_gather, y, x, n_q, codes, scales, ra, st, sy)
                                 : gqr_t<T, QBITS, RBIN, 4, false>(pc, n_gather, y, x, n_q, codes, scales, ra, st, sy);
  }
  return cudaErrorNotSupported;
}

template <typename T>
cudaError_t gqr_d(const Pieces& pc, int64_t n_gather, void* y, const void* x, int64_t n_q, int qbits, uint8_t* codes,
                  float* scales, const RedArgs& ra, int rbits, cudaStream_t st, const SyncArgs& sy) {
  if (qbits == 4)
    return rbits == 4 ? gqr_g<T, 4, 4>(pc, n_gather, y, x, n_q, codes, scales, ra, st, sy)
                      : gqr_g<T, 4, 8>(pc, n_gather, y, x, n_q, codes, scales, ra, st, sy);
  return rbits == 4 ? gqr_g<T, 8, 4>(pc, n_gather, y, x, n_q, codes, scales, ra, st, sy)
                    : gqr_g<T, 8, 8>(pc, n_gather, y, x, n_q, codes, scales, ra, st, sy);
}

}  // namespace

cudaError_t launch_reduce(int g, const uint8_t* const* codes, const float* const* scales,
                          int64_t n, int bits_in, int block, int bits_out, uint8_t* out_codes,
                          float* out_scales, float* out_f32, int accumulate, cudaStream_t st,
                          const SyncArgs* sync) {
  const SyncArgs sy = sync ? *sync : SyncArgs{};
  if (n == 0 && !sync) return cudaSuccess;
  RedArgs a{};
  for (int p = 0; p < g; ++p) {
    a.c[p] = codes[p];
    a.s[p] = scales[p];
  }
  a.g = g;
  a.accumulate = accumulate;
  a.n = n;
  a.oc = out_codes;
  a.os = out_scales;
  a.of = out_f32;
  {
    const cudaError_t e = tiles_reduce(g, codes, scales, n, bits_in, block, bits_out, out_codes, out_scales, out_f32,
                                       accumulate, st, sy);
    if (e != cudaErrorNotSupported) return e;
  }
  if (bits_out == 0) {
    int log2b = 0;
    while ((1 << log2b) < block) ++log2b;
    return bits_in == 8 ? f32_g<8>(a, log2b, st, sy) : f32_g<4>(a, log2b, st, sy);
  }
  switch (block) {
    case 32: return requant_b<32>(a, bits_in, bits_out, st, sy);
    case 64: return requant_b<64>(a, bits_in, bits_out, st, sy);
    case 128: return requant_b<128>(a, bits_in, bits_out, st, sy);
    case 256: return requant_b<256>(a, bits_in, bits_out, st, sy);
    case 512: return requant_b<512>(a, bits_in, bits_out, st, sy);
    case 1024: return requant_b<1024>(a, bits_in, bits_out, st, sy);
    case 2048: return requant_b<2048>(a, bits_in, bits_out, st, sy);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hz

namespace hz {

bool gather_quantize_reduce_supported(int gather_bits, hz_dtype out_dt, int g, int red_bits) {
  return gather_bits == 8 && out_dt == HZ_BF16 && (g == 2 || g == 4) && (red_bits == 4 || red_bits == 8);
}

cudaError_t launch_gather_quantize_reduce(const Pieces& pc, int64_t n_gather, void* y, const void* x, hz_dtype dt,
                                          int64_t n_q, int qbits, uint8_t* codes, float* scales, int g,
                                          const uint8_t* const* rc, const float* const* rs, int64_t rn, int rbits,
                                          float* shard, int acc, cudaStream_t st, const SyncArgs& sy) {
  RedArgs ra{};
  for (int p = 0; p < g; ++p) {
    ra.c[p] = rc[p];
    ra.s[p] = rs[p];
  }
  ra.g = g;
  ra.accumulate = acc;
  ra.n = rn;
  ra.of = shard;
  switch (dt) {
    case HZ_F32: return gqr_d<float>(pc, n_gather, y, x, n_q, qbits, codes, scales, ra, rbits, st, sy);
    case HZ_BF16: return gqr_d<__nv_bfloat16>(pc, n_gather, y, x, n_q, qbits, codes, scales, ra, rbits, st, sy);
    case HZ_F16: return gqr_d<__half>(pc, n_gather, y, x, n_q, qbits, codes, scales, ra, rbits, st, sy);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hz
