// sm_100a codec kernels of the hierarchical ZeRO++ hot path.
//
//   k_quantize   (A2 / A7, O4-O5)  x (bf16|fp16|fp32) -> int8|int4 codes + fp32 scale / block
//   k_dequantize (A5 / A6, O6)     codes + scales -> bf16|fp16|fp32
//   k_reduce     (A9 / A10, O9)    g coded chunks -> fp32 sum (ascending p, no FMA)
//                                  -> requantized codes (next level) or fp32 shard (+=)
//
// All three are HBM-streaming kernels (no dense contraction, so no tensor cores;
// DESIGN.md §6).  Data movement: every lane owns 8 consecutive elements per
// "sub-chunk" and the lanes of a warp own consecutive sub-chunks, so every load
// and store instruction of a warp touches one contiguous span (16-byte bf16
// loads, 8/4-byte code stores, 16-byte bf16 stores).  A quantization block of B
// elements is owned by LPB = min(32, B/8) lanes; its absmax is a shuffle-xor
// reduction inside those lanes.  Each warp issues the loads of U independent
// warp-steps before consuming any (memory-level parallelism), and the grid is a
// grid-stride loop sized to SMs x resident CTAs.
//
// Exactness (parity with the oracle): bf16/fp16 -> fp32 widening
// is exact; scale = __fdiv_rn(am, qmax), inv = __fdiv_rn(qmax, am),
// code = __float2int_rn(__fmul_rn(x, inv)); x_hat = __fmul_rn(code, scale);
// sums use __fadd_rn (never contracted into FMA; the library is also built with
// --fmad=false).  Output bf16/fp16 conversions are RNE.

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <mutex>
#include <unordered_map>

#include "hz_internal.h"

namespace hz {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr float kTiny = 0x1p-100f;   // R3: am < 2^-100 -> scale 0, codes 0
constexpr int kThreads = 256;

template <int B>
struct Geo {
  static constexpr int LPB = B >= 256 ? 32 : B / 8;     // lanes per quantization block
  static constexpr int NSUB = B >= 256 ? B / 256 : 1;   // 8-element sub-chunks per lane per block
  static constexpr int BPW = 32 / LPB;                  // blocks per warp step
  static constexpr int SUBSTRIDE = LPB * 8;             // elements between a lane's sub-chunks
};

template <int BITS>
struct QMax;
template <>
struct QMax<8> { static constexpr int v = 127; };
template <>
struct QMax<4> { static constexpr int v = 7; };

// ------------------------------------------------------------ 8-element input
template <typename T>
struct In8;

template <>
struct In8<float> {
  uint4 r[2];
  __device__ __forceinline__ void load(const float* p) {
    r[0] = __ldg(reinterpret_cast<const uint4*>(p));
    r[1] = __ldg(reinterpret_cast<const uint4*>(p) + 1);
  }
  __device__ __forceinline__ void get(float (&v)[8]) const {
    v[0] = __uint_as_float(r[0].x); v[1] = __uint_as_float(r[0].y);
    v[2] = __uint_as_float(r[0].z); v[3] = __uint_as_float(r[0].w);
    v[4] = __uint_as_float(r[1].x); v[5] = __uint_as_float(r[1].y);
    v[6] = __uint_as_float(r[1].z); v[7] = __uint_as_float(r[1].w);
  }
};

template <>
struct In8<__nv_bfloat16> {
  uint4 r;
  __device__ __forceinline__ void load(const __nv_bfloat16* p) {
    r = __ldg(reinterpret_cast<const uint4*>(p));
  }
  __device__ __forceinline__ void get(float (&v)[8]) const {
    // bf16 -> fp32 is a 16-bit left shift: exact (subnormals included).
    v[0] = __uint_as_float(r.x << 16); v[1] = __uint_as_float(r.x & 0xffff0000u);
    v[2] = __uint_as_float(r.y << 16); v[3] = __uint_as_float(r.y & 0xffff0000u);
    v[4] = __uint_as_float(r.z << 16); v[5] = __uint_as_float(r.z & 0xffff0000u);
    v[6] = __uint_as_float(r.w << 16); v[7] = __uint_as_float(r.w & 0xffff0000u);
  }
};

template <>
struct In8<__half> {
  uint4 r;
  __device__ __forceinline__ void load(const __half* p) {
    r = __ldg(reinterpret_cast<const uint4*>(p));
  }
  __device__ __forceinline__ void get(float (&v)[8]) const {
    const unsigned w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h = *reinterpret_cast<const __half2*>(&w[i]);
      float2 f = __half22float2(h);   // exact
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  }
};

// ------------------------------------------------------------ 8-element codes
template <int BITS>
struct Codes8;

template <>
struct Codes8<8> {
  uint2 r;
  __device__ __forceinline__ void load(const uint8_t* p) { r = __ldg(reinterpret_cast<const uint2*>(p)); }
  __device__ __forceinline__ void store(uint8_t* p) const { *reinterpret_cast<uint2*>(p) = r; }
  __device__ __forceinline__ int code(int i) const {
    const unsigned w = i < 4 ? r.x : r.y;
    return static_cast<int>(w << (24 - 8 * (i & 3))) >> 24;   // sign-extend byte
  }
  __device__ __forceinline__ void set(const int (&c)[8]) {
    r.x = (c[0] & 0xff) | ((c[1] & 0xff) << 8) | ((c[2] & 0xff) << 16) | ((unsigned)(c[3] & 0xff) << 24);
    r.y = (c[4] & 0xff) | ((c[5] & 0xff) << 8) | ((c[6] & 0xff) << 16) | ((unsigned)(c[7] & 0xff) << 24);
  }
};

template <>
struct Codes8<4> {
  unsigned r;
  __device__ __forceinline__ void load(const uint8_t* p) { r = __ldg(reinterpret_cast<const unsigned*>(p)); }
  __device__ __forceinline__ void store(uint8_t* p) const { *reinterpret_cast<unsigned*>(p) = r; }
  __device__ __forceinline__ int code(int i) const {
    return static_cast<int>(r << (28 - 4 * i)) >> 28;            // sign-extend nibble
  }
  __device__ __forceinline__ void set(const int (&c)[8]) {
    unsigned v = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) v |= (unsigned)(c[i] & 0xf) << (4 * i);   // even element low (R4)
    r = v;
  }
};

// ------------------------------------------------------------------- codec math
template <int BITS>
__device__ __forceinline__ void quant_params(float am, float& scale, float& inv) {
  constexpr float qmax = static_cast<float>(QMax<BITS>::v);
  if (am >= kTiny) {
    scale = __fdiv_rn(am, qmax);
    inv = __fdiv_rn(qmax, am);
  } else {
    scale = 0.f;
    inv = 0.f;
  }
}

template <int BITS>
__device__ __forceinline__ int qcode(float v, float inv) {
  constexpr int qmax = QMax<BITS>::v;
  int c = __float2int_rn(__fmul_rn(v, inv));
  return max(-qmax, min(qmax, c));
}

template <int LPB>
__device__ __forceinline__ float group_max(float v) {
#pragma unroll
  for (int o = LPB / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// ------------------------------------------------------------------ output store
template <typename TO>
struct Out8;

template <>
struct Out8<float> {
  __device__ __forceinline__ static void store(float* p, const float (&v)[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};

template <>
struct Out8<__nv_bfloat16> {
  __device__ __forceinline__ static void store(__nv_bfloat16* p, const float (&v)[8]) {
    uint4 o;
    unsigned w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);   // RNE
      w[i] = *reinterpret_cast<unsigned*>(&h);
    }
    o.x = w[0]; o.y = w[1]; o.z = w[2]; o.w = w[3];
    *reinterpret_cast<uint4*>(p) = o;
  }
};

template <>
struct Out8<__half> {
  __device__ __forceinline__ static void store(__half* p, const float (&v)[8]) {
    uint4 o;
    unsigned w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<unsigned*>(&h);
    }
    o.x = w[0]; o.y = w[1]; o.z = w[2]; o.w = w[3];
    *reinterpret_cast<uint4*>(p) = o;
  }
};

// =============================================================== k_quantize
// One warp step = BPW blocks = max(B, 256) contiguous elements.  A warp owns U
// consecutive steps per iteration of the grid-stride loop.
template <typename T, int B, int BITS, int U>
__global__ void __launch_bounds__(kThreads) k_quantize(const T* __restrict__ x, int64_t nblocks,
                                                       uint8_t* __restrict__ codes,
                                                       float* __restrict__ scales) {
  using G = Geo<B>;
  const int lane = threadIdx.x & 31;
  const int lb = lane / G::LPB;
  const int ll = lane % G::LPB;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * kThreads) >> 5;
  const int64_t nsteps = (nblocks + G::BPW - 1) / G::BPW;

  for (int64_t s0 = warp * U; s0 < nsteps; s0 += nwarps * U) {
    In8<T> raw[U][G::NSUB];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t blk = (s0 + u) * G::BPW + lb;
      if (s0 + u < nsteps && blk < nblocks) {
#pragma unroll
        for (int k = 0; k < G::NSUB; ++k) raw[u][k].load(x + blk * B + k * G::SUBSTRIDE + ll * 8);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t blk = (s0 + u) * G::BPW + lb;
      const bool valid = (s0 + u < nsteps) && blk < nblocks;
      float v[G::NSUB][8];
      float am = 0.f;
#pragma unroll
      for (int k = 0; k < G::NSUB; ++k) {
        if (valid) {
          raw[u][k].get(v[k]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) v[k][i] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) am = fmaxf(am, fabsf(v[k][i]));
      }
      am = group_max<G::LPB>(am);
      float scale, inv;
      quant_params<BITS>(am, scale, inv);
      if (valid) {
#pragma unroll
        for (int k = 0; k < G::NSUB; ++k) {
          int c[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) c[i] = qcode<BITS>(v[k][i], inv);
          Codes8<BITS> out;
          out.set(c);
          out.store(codes + (blk * B + k * G::SUBSTRIDE + ll * 8) * BITS / 8);
        }
        if (ll == 0) scales[blk] = scale;
      }
    }
  }
}

// ============================================================= k_dequantize
// Elementwise: one "unit" = 8 consecutive elements; the lanes of a warp own 32
// consecutive units per instruction; U instructions per iteration.
template <int BITS, typename TO, int U>
__global__ void __launch_bounds__(kThreads) k_dequantize(const uint8_t* __restrict__ codes,
                                                         const float* __restrict__ scales,
                                                         int64_t nunits, int log2b,
                                                         TO* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * kThreads) >> 5;
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
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __fmul_rn(static_cast<float>(raw[u].code(i)), sc[u]);
        Out8<TO>::store(y + unit * 8, v);
      }
    }
  }
}

// ================================================================= k_reduce
struct RedArgs {
  const uint8_t* c[kMaxG];
  const float* s[kMaxG];
  int g;
  int accumulate;
  int64_t nblocks;
  uint8_t* oc;
  float* os;
  float* of;
};

// GT > 0: exactly GT inputs, all loads of a step issued before the sums.
// GT == 0: runtime a.g inputs, one input at a time.
template <int B, int BIN, int BOUT, int GT, int U>
__global__ void __launch_bounds__(kThreads) k_reduce(const __grid_constant__ RedArgs a) {
  using G = Geo<B>;
  const int lane = threadIdx.x & 31;
  const int lb = lane / G::LPB;
  const int ll = lane % G::LPB;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * kThreads) >> 5;
  const int64_t nsteps = (a.nblocks + G::BPW - 1) / G::BPW;
  constexpr int GP = GT > 0 ? GT : 1;

  for (int64_t s0 = warp * U; s0 < nsteps; s0 += nwarps * U) {
    float acc[U][G::NSUB][8];
    if constexpr (GT > 0) {
      Codes8<BIN> raw[U][GP][G::NSUB];
      float sc[U][GP];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t blk = (s0 + u) * G::BPW + lb;
        if (s0 + u < nsteps && blk < a.nblocks) {
#pragma unroll
          for (int p = 0; p < GP; ++p) {
#pragma unroll
            for (int k = 0; k < G::NSUB; ++k)
              raw[u][p][k].load(a.c[p] + (blk * B + k * G::SUBSTRIDE + ll * 8) * BIN / 8);
            sc[u][p] = __ldg(a.s[p] + blk);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int k = 0; k < G::NSUB; ++k) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float s = __fmul_rn(static_cast<float>(raw[u][0][k].code(i)), sc[u][0]);
#pragma unroll
            for (int p = 1; p < GP; ++p)
              s = __fadd_rn(s, __fmul_rn(static_cast<float>(raw[u][p][k].code(i)), sc[u][p]));
            acc[u][k][i] = s;
          }
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < G::NSUB; ++k)
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[u][k][i] = 0.f;
      for (int p = 0; p < a.g; ++p) {
        Codes8<BIN> raw[U][G::NSUB];
        float sc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t blk = (s0 + u) * G::BPW + lb;
          if (s0 + u < nsteps && blk < a.nblocks) {
#pragma unroll
            for (int k = 0; k < G::NSUB; ++k)
              raw[u][k].load(a.c[p] + (blk * B + k * G::SUBSTRIDE + ll * 8) * BIN / 8);
            sc[u] = __ldg(a.s[p] + blk);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int k = 0; k < G::NSUB; ++k)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float xh = __fmul_rn(static_cast<float>(raw[u][k].code(i)), sc[u]);
              acc[u][k][i] = p == 0 ? xh : __fadd_rn(acc[u][k][i], xh);
            }
      }
    }

#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t blk = (s0 + u) * G::BPW + lb;
      const bool valid = (s0 + u < nsteps) && blk < a.nblocks;
      if constexpr (BOUT == 0) {
        if (valid) {
#pragma unroll
          for (int k = 0; k < G::NSUB; ++k) {
            float* dst = a.of + blk * B + k * G::SUBSTRIDE + ll * 8;
            float v[8];
            if (a.accumulate) {
              const float4 o0 = reinterpret_cast<const float4*>(dst)[0];
              const float4 o1 = reinterpret_cast<const float4*>(dst)[1];
              const float old[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
              for (int i = 0; i < 8; ++i) v[i] = __fadd_rn(old[i], acc[u][k][i]);
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i) v[i] = acc[u][k][i];
            }
            Out8<float>::store(dst, v);
          }
        }
      } else {
        float am = 0.f;
#pragma unroll
        for (int k = 0; k < G::NSUB; ++k)
#pragma unroll
          for (int i = 0; i < 8; ++i) am = fmaxf(am, valid ? fabsf(acc[u][k][i]) : 0.f);
        am = group_max<G::LPB>(am);
        float scale, inv;
        quant_params<BOUT>(am, scale, inv);
        if (valid) {
#pragma unroll
          for (int k = 0; k < G::NSUB; ++k) {
            int c[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) c[i] = qcode<BOUT>(acc[u][k][i], inv);
            Codes8<BOUT> out;
            out.set(c);
            out.store(a.oc + (blk * B + k * G::SUBSTRIDE + ll * 8) * BOUT / 8);
          }
          if (ll == 0) a.os[blk] = scale;
        }
      }
    }
  }
}

// =============================================================== launch helpers
int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 148;
  }
  return cached[dev];
}

int resident_ctas(const void* kernel) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(kernel);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, kThreads, 0) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = 1;
  }
  cache[kernel] = n;
  return n;
}

int64_t grid_for(const void* kernel, int64_t warp_tasks) {
  const int64_t need = (warp_tasks + (kThreads / 32) - 1) / (kThreads / 32);
  const int64_t cap = static_cast<int64_t>(sm_count()) * resident_ctas(kernel);
  int64_t gsz = need < cap ? need : cap;
  return gsz < 1 ? 1 : gsz;
}

constexpr int kUQ = 4;   // warp steps in flight per warp (quantize)
constexpr int kUD = 4;   // 8-element units in flight per lane (dequantize)
constexpr int kUR = 2;   // warp steps in flight per warp (reduce)
// Blocks larger than 256 already give each lane NSUB = B/256 independent loads per
// step; keep one step in flight there so registers do not spill.
constexpr int uq(int B) { return B > 256 ? 1 : kUQ; }
constexpr int ur(int B) { return B > 256 ? 1 : kUR; }

template <typename T, int B, int BITS>
cudaError_t quantize_t(const void* x, int64_t n, uint8_t* codes, float* scales, cudaStream_t st) {
  const int64_t nblocks = n / B;
  const int64_t nsteps = (nblocks + Geo<B>::BPW - 1) / Geo<B>::BPW;
  constexpr int U = uq(B);
  auto kern = k_quantize<T, B, BITS, U>;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), (nsteps + U - 1) / U);
  kern<<<static_cast<unsigned>(grid), kThreads, 0, st>>>(static_cast<const T*>(x), nblocks, codes, scales);
  return cudaGetLastError();
}

template <typename T, int B>
cudaError_t quantize_b(const void* x, int64_t n, int bits, uint8_t* c, float* s, cudaStream_t st) {
  return bits == 8 ? quantize_t<T, B, 8>(x, n, c, s, st) : quantize_t<T, B, 4>(x, n, c, s, st);
}

template <typename T>
cudaError_t quantize_d(const void* x, int64_t n, int bits, int block, uint8_t* c, float* s,
                       cudaStream_t st) {
  switch (block) {
    case 32: return quantize_b<T, 32>(x, n, bits, c, s, st);
    case 64: return quantize_b<T, 64>(x, n, bits, c, s, st);
    case 128: return quantize_b<T, 128>(x, n, bits, c, s, st);
    case 256: return quantize_b<T, 256>(x, n, bits, c, s, st);
    case 512: return quantize_b<T, 512>(x, n, bits, c, s, st);
    case 1024: return quantize_b<T, 1024>(x, n, bits, c, s, st);
    case 2048: return quantize_b<T, 2048>(x, n, bits, c, s, st);
  }
  return cudaErrorInvalidValue;
}

template <int BITS, typename TO>
cudaError_t dequantize_t(const uint8_t* codes, const float* scales, int64_t n, int block, void* y,
                         cudaStream_t st) {
  const int64_t nunits = n / 8;
  int log2b = 0;
  while ((1 << log2b) < block) ++log2b;
  auto kern = k_dequantize<BITS, TO, kUD>;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), (nunits + 32 * kUD - 1) / (32 * kUD));
  kern<<<static_cast<unsigned>(grid), kThreads, 0, st>>>(codes, scales, nunits, log2b, static_cast<TO*>(y));
  return cudaGetLastError();
}

template <int B, int BIN, int BOUT, int GT>
cudaError_t reduce_t(const RedArgs& a, cudaStream_t st) {
  const int64_t nsteps = (a.nblocks + Geo<B>::BPW - 1) / Geo<B>::BPW;
  constexpr int U = ur(B);
  auto kern = k_reduce<B, BIN, BOUT, GT, U>;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), (nsteps + U - 1) / U);
  kern<<<static_cast<unsigned>(grid), kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

template <int B, int BIN, int BOUT>
cudaError_t reduce_g(const RedArgs& a, cudaStream_t st) {
  // Fully unrolled input prefetch for the common group sizes; large blocks with
  // many inputs use the one-input-at-a-time loop (register budget).
  switch (a.g) {
    case 1: return reduce_t<B, BIN, BOUT, 1>(a, st);
    case 2: return reduce_t<B, BIN, BOUT, 2>(a, st);
    case 4: return B >= 1024 ? reduce_t<B, BIN, BOUT, 0>(a, st) : reduce_t<B, BIN, BOUT, 4>(a, st);
    case 8: return B >= 512 ? reduce_t<B, BIN, BOUT, 0>(a, st) : reduce_t<B, BIN, BOUT, 8>(a, st);
    default: return reduce_t<B, BIN, BOUT, 0>(a, st);
  }
}

template <int B, int BIN>
cudaError_t reduce_o(const RedArgs& a, int bits_out, cudaStream_t st) {
  switch (bits_out) {
    case 0: return reduce_g<B, BIN, 0>(a, st);
    case 4: return reduce_g<B, BIN, 4>(a, st);
    case 8: return reduce_g<B, BIN, 8>(a, st);
  }
  return cudaErrorInvalidValue;
}

template <int B>
cudaError_t reduce_i(const RedArgs& a, int bits_in, int bits_out, cudaStream_t st) {
  return bits_in == 8 ? reduce_o<B, 8>(a, bits_out, st) : reduce_o<B, 4>(a, bits_out, st);
}

}  // namespace

cudaError_t launch_quantize(const void* x, hz_dtype dt, int64_t n, int bits, int block,
                            uint8_t* codes, float* scales, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  switch (dt) {
    case HZ_F32: return quantize_d<float>(x, n, bits, block, codes, scales, st);
    case HZ_BF16: return quantize_d<__nv_bfloat16>(x, n, bits, block, codes, scales, st);
    case HZ_F16: return quantize_d<__half>(x, n, bits, block, codes, scales, st);
  }
  return cudaErrorInvalidValue;
}

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

cudaError_t launch_reduce(int g, const uint8_t* const* codes, const float* const* scales,
                          int64_t n, int bits_in, int block, int bits_out, uint8_t* out_codes,
                          float* out_scales, float* out_f32, int accumulate, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  RedArgs a{};
  for (int p = 0; p < g; ++p) {
    a.c[p] = codes[p];
    a.s[p] = scales[p];
  }
  a.g = g;
  a.accumulate = accumulate;
  a.nblocks = n / block;
  a.oc = out_codes;
  a.os = out_scales;
  a.of = out_f32;
  switch (block) {
    case 32: return reduce_i<32>(a, bits_in, bits_out, st);
    case 64: return reduce_i<64>(a, bits_in, bits_out, st);
    case 128: return reduce_i<128>(a, bits_in, bits_out, st);
    case 256: return reduce_i<256>(a, bits_in, bits_out, st);
    case 512: return reduce_i<512>(a, bits_in, bits_out, st);
    case 1024: return reduce_i<1024>(a, bits_in, bits_out, st);
    case 2048: return reduce_i<2048>(a, bits_in, bits_out, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hz
