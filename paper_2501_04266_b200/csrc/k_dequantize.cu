// k_dequantize (A5 forward / A6 backward; oracle O6): codes + fp32 scales ->
// bf16 | fp16 | fp32, x_hat = fl(code * scale), RNE narrowing.  Every rank,
// the owner of a shard included, dequantizes the whole gathered layer from the
// codes (R9), so the layer is bit-identical on all ranks.  Paper: "quantizer and
// dequantizer operators from ZeRO++".
//
// Elementwise: a unit = 8 consecutive elements (8/4 code bytes in, one 16-byte
// bf16 store out); the lanes of a warp own 32 consecutive units per instruction
// (contiguous spans); each lane keeps U units in flight.
#include "codec.cuh"

namespace hz {
namespace {

using namespace dev;

template <int BITS, typename TO, int U>
__global__ void __launch_bounds__(kThreads) k_dequantize(const uint8_t* __restrict__ codes,
                                                         const float* __restrict__ scales,
                                                         int64_t nunits, int log2b,
                                                         TO* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = global_warp();
  const int64_t nwarps = num_warps();
  for (int64_t base = warp * 32 * U; base < nunits; base += nwarps * 32 * U) {
    Codes8<BITS> raw[U];
    float sc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t unit = base + u * 32 + lane;
      if (unit < nunits) {
        raw[u].load(codes + unit * BITS);
        sc[u] = __ldg(scales + ((unit * 8) >> log2b));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t unit = base + u * 32 + lane;
      if (unit < nunits) {
        float c[8], v[8];
        raw[u].decode(c);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __fmul_rn(c[i], sc[u]);
        Out8<TO>::store(y + unit * 8, v);
      }
    }
  }
}

constexpr int kU = 4;   // units in flight per lane (HZ_TUNE deq_u: 2, 4, 8, 16)

template <int BITS, typename TO, int U>
cudaError_t dequantize_u(const uint8_t* codes, const float* scales, int64_t nunits, int log2b, void* y,
                         cudaStream_t st) {
  auto kern = k_dequantize<BITS, TO, U>;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), (nunits + 32 * U - 1) / (32 * U));
  kern<<<static_cast<unsigned>(grid), kThreads, 0, st>>>(codes, scales, nunits, log2b, static_cast<TO*>(y));
  return cudaGetLastError();
}

template <int BITS, typename TO>
cudaError_t dequantize_t(const uint8_t* codes, const float* scales, int64_t n, int block, void* y,
                         cudaStream_t st) {
  const int64_t nunits = n / 8;
  int log2b = 0;
  while ((1 << log2b) < block) ++log2b;
  switch (tune_param("deq_u", kU)) {
    case 2: return dequantize_u<BITS, TO, 2>(codes, scales, nunits, log2b, y, st);
    case 8: return dequantize_u<BITS, TO, 8>(codes, scales, nunits, log2b, y, st);
    case 16: return dequantize_u<BITS, TO, 16>(codes, scales, nunits, log2b, y, st);
    default: return dequantize_u<BITS, TO, kU>(codes, scales, nunits, log2b, y, st);
  }
}

}  // namespace

cudaError_t launch_dequantize(const uint8_t* codes, const float* scales, int64_t n, int bits,
                              int block, void* y, hz_dtype out_dt, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  if (bits == 8) {
    switch (out_dt) {
      case HZ_F32: return dequantize_t<8, float>(codes, scales, n, block, y, st);
      case HZ_BF16: return dequantize_t<8, __nv_bfloat16>(codes, scales, n, block, y, st);
      case HZ_F16: return dequantize_t<8, __half>(codes, scales, n, block, y, st);
    }
  } else {
    switch (out_dt) {
      case HZ_F32: return dequantize_t<4, float>(codes, scales, n, block, y, st);
      case HZ_BF16: return dequantize_t<4, __nv_bfloat16>(codes, scales, n, block, y, st);
      case HZ_F16: return dequantize_t<4, __half>(codes, scales, n, block, y, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace hz
