// The quantize loop of k_quantize (see k_quantize.cu), shared with the dual kernel
// (k_gather_quantize) and the backward triple kernel (k_reduce.cu,
// k_gather_quantize_reduce): warp `warp` of `nwarps` processes its share of the blocks.
// Internal header.
#pragma once

#include "codec.cuh"

namespace hz {
namespace dev {

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
template <>
struct OutOf<4> { using E = EmitF32Bulk; };   // fp32 round trip, no accumulate, TMA stores
template <>
struct OutOf<5> { using E = EmitOutBulk<__nv_bfloat16>; };   // bf16 round trip, TMA stores
template <>
struct OutOf<6> { using E = EmitOutBulk<__half>; };          // fp16 round trip, TMA stores

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
        if constexpr (OUT == 1 || OUT == 2 || OUT == 5 || OUT == 6) {
          if (valid) {   // warp-uniform for B = 256 (the round trip's block)
            float xh[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) xh[i] = __fmul_rn(__fsub_rn(__uint_as_float(b[i]), kMagic), scale);
            emit(blk * B + k * G::SUBSTRIDE + ll * 8, lane, xh);
          }
        } else if constexpr (OUT == 3 || OUT == 4) {
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

}  // namespace dev
}  // namespace hz
