// The level-reduce pieces shared by k_reduce.cu's kernels and the backward triple
// kernel (k_gather_quantize_reduce): the argument block, the wide code loads and the
// fp32-output reduce loop.  Internal header.
#pragma once

#include "codec.cuh"

namespace hz {
namespace dev {

constexpr int kMaxGIn = kMaxG;

struct RedArgs {
  const uint8_t* c[kMaxG];
  const float* s[kMaxG];
  int g;
  int accumulate;
  int64_t n;          // elements
  uint8_t* oc;
  float* os;
  float* of;
};

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

// The fp32-output reduce (k_reduce_f32's body): warp `warp` of `nwarps` reduces its
// grid-stride share of the units; `st` = this warp's 32*G float4 staging granules.
template <int BIN>
__host__ __device__ constexpr int red_granules() { return Wide<BIN>::E / 4; }

template <int BIN, int GT, int U, bool ACC>
__device__ __forceinline__ void reduce_f32_loop(const RedArgs& a, int log2b, float4* st, int64_t warp, int64_t nwarps) {
  constexpr int E = Wide<BIN>::E;
  constexpr int G = E / 4;                         // float4 granules per lane per unit
  const int lane = threadIdx.x & 31;
  const int64_t nunits = a.n / E;
  constexpr int GP = GT > 0 ? GT : 1;
  for (int64_t base = warp * 32 * U; base < nunits; base += nwarps * 32 * U) {
    float acc[U][E];
    float4 old[ACC ? U : 1][G];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t chunk = base + u * 32;            // first unit of this warp chunk
      if (ACC && chunk < nunits) {
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const int64_t g4 = chunk * G + k * 32 + lane;   // float4 index, contiguous per k
          if (g4 < nunits * G) old[u][k] = reinterpret_cast<const float4*>(a.of)[g4];
        }
      }
    }
    if constexpr (GT > 0) {
      Wide<BIN> raw[U][GP];
      float sc[U][GP];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t unit = base + u * 32 + lane;
#pragma unroll
        for (int p = 0; p < GP; ++p) {
          sc[u][p] = 0.f;
          raw[u][p].r = make_uint2(0u, 0u);
          if (unit < nunits) {
            raw[u][p].load(a.c[p] + unit * 8);
            sc[u][p] = HZ_PEER_LD(a.s[p] + ((unit * E) >> log2b));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float c[E];
        raw[u][0].decode(c);
#pragma unroll
        for (int i = 0; i < E; ++i) acc[u][i] = __fmul_rn(c[i], sc[u][0]);
#pragma unroll
        for (int p = 1; p < GP; ++p) {
          raw[u][p].decode(c);
#pragma unroll
          for (int i = 0; i < E; ++i) acc[u][i] = __fadd_rn(acc[u][i], __fmul_rn(c[i], sc[u][p]));
        }
      }
    } else {
      for (int p = 0; p < a.g; ++p) {
        Wide<BIN> raw[U];
        float sc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t unit = base + u * 32 + lane;
          sc[u] = 0.f;
          raw[u].r = make_uint2(0u, 0u);
          if (unit < nunits) {
            raw[u].load(a.c[p] + unit * 8);
            sc[u] = HZ_PEER_LD(a.s[p] + ((unit * E) >> log2b));
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float c[E];
          raw[u].decode(c);
#pragma unroll
          for (int i = 0; i < E; ++i) {
            const float xh = __fmul_rn(c[i], sc[u]);
            acc[u][i] = p == 0 ? xh : __fadd_rn(acc[u][i], xh);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t chunk = base + u * 32;
      if (chunk >= nunits) break;                      // warp-uniform
      // lane's E sums -> granules lane*G + j (swizzled), then read back granule k*32 + lane
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int gi = lane * G + j;
        st[gi ^ ((gi >> 3) & (G - 1))] = make_float4(acc[u][4 * j], acc[u][4 * j + 1], acc[u][4 * j + 2], acc[u][4 * j + 3]);
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < G; ++k) {
        const int gi = k * 32 + lane;
        float4 o = st[gi ^ ((gi >> 3) & (G - 1))];
        const int64_t g4 = chunk * G + gi;
        if (g4 < nunits * G) {
          if constexpr (ACC) {
            o.x = __fadd_rn(old[u][k].x, o.x);
            o.y = __fadd_rn(old[u][k].y, o.y);
            o.z = __fadd_rn(old[u][k].z, o.z);
            o.w = __fadd_rn(old[u][k].w, o.w);
          }
          reinterpret_cast<float4*>(a.of)[g4] = o;
        }
      }
      __syncwarp();
    }
  }
}

}  // namespace dev
}  // namespace hz
