// Step tail (oracle/optim.py):
//   k_adamw        AdamW on the optimizer shard (fp32 master, m, v):
//                  one pass reads g, theta, m, v and writes theta', m', v' and the
//                  updated weights in the parameter dtype (30 B/element, HBM-bound).
//   k_gather_copy  post-update all-gather over NVLink: the members' updated
//                  shards are read straight from their pools (interleaved tiles, as
//                  the gather-dequantize) into the rank's primary range.
//   k_sum_f32      one level of the paper-literal allreduce (A10 option):
//                  out = ((x_0 + x_1) + ...) + x_{g-1}, fp32, ascending member digit
//                  (the inputs may be peer-mapped; g == 1 is a copy).
// Arithmetic: one IEEE rounding per operation in the oracle's order (__fmul_rn,
// __fadd_rn, __fsub_rn, __fsqrt_rn, __fdiv_rn; no FMA).
#include "codec.cuh"

namespace hz {
namespace {

using namespace dev;

template <typename TO>
__device__ __forceinline__ void store4(TO* p, const float (&v)[4]);
template <>
__device__ __forceinline__ void store4<float>(float* p, const float (&v)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* p, const float (&v)[4]) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
  *reinterpret_cast<uint2*>(p) = make_uint2(*reinterpret_cast<unsigned*>(&a), *reinterpret_cast<unsigned*>(&b));
}
template <>
__device__ __forceinline__ void store4<__half>(__half* p, const float (&v)[4]) {
  __half2 a = __floats2half2_rn(v[0], v[1]), b = __floats2half2_rn(v[2], v[3]);
  *reinterpret_cast<uint2*>(p) = make_uint2(*reinterpret_cast<unsigned*>(&a), *reinterpret_cast<unsigned*>(&b));
}

template <typename TO, int U>
__global__ void __launch_bounds__(kThreads) k_adamw(const float* __restrict__ g, float* __restrict__ th,
                                                    float* __restrict__ m, float* __restrict__ v,
                                                    TO* __restrict__ out, int64_t n4, AdamW hp,
                                                    const __grid_constant__ SyncArgs sy) {
  if (!sync_wait(sy)) return;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
  const int64_t nth = static_cast<int64_t>(gridDim.x) * kThreads;
  for (int64_t base = tid; base < n4; base += nth * U) {
    float4 G[U], T[U], M[U], V[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * nth;
      if (i < n4) {
        G[u] = reinterpret_cast<const float4*>(g)[i];
        T[u] = reinterpret_cast<const float4*>(th)[i];
        M[u] = reinterpret_cast<const float4*>(m)[i];
        V[u] = reinterpret_cast<const float4*>(v)[i];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * nth;
      if (i >= n4) continue;
      const float gg[4] = {G[u].x, G[u].y, G[u].z, G[u].w};
      const float tt[4] = {T[u].x, T[u].y, T[u].z, T[u].w};
      const float mm[4] = {M[u].x, M[u].y, M[u].z, M[u].w};
      const float vv[4] = {V[u].x, V[u].y, V[u].z, V[u].w};
      float mo[4], vo[4], to[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        mo[k] = __fadd_rn(__fmul_rn(hp.b1, mm[k]), __fmul_rn(hp.omb1, gg[k]));
        vo[k] = __fadd_rn(__fmul_rn(hp.b2, vv[k]), __fmul_rn(__fmul_rn(hp.omb2, gg[k]), gg[k]));
        const float t1 = __fsub_rn(tt[k], __fmul_rn(hp.lr_wd, tt[k]));
        const float den = __fadd_rn(__fdiv_rn(__fsqrt_rn(vo[k]), hp.sqrt_bc2), hp.eps);
        to[k] = __fsub_rn(t1, __fmul_rn(hp.step, __fdiv_rn(mo[k], den)));
      }
      reinterpret_cast<float4*>(m)[i] = make_float4(mo[0], mo[1], mo[2], mo[3]);
      reinterpret_cast<float4*>(v)[i] = make_float4(vo[0], vo[1], vo[2], vo[3]);
      reinterpret_cast<float4*>(th)[i] = make_float4(to[0], to[1], to[2], to[3]);
      store4<TO>(out + i * 4, to);
    }
  }
  sync_signal(sy);
}

// 16-byte pieces copy: pieces of len bytes (a multiple of 16) interleaved by warp
// tile; piece j -> out + j * len.
template <int U>
__global__ void __launch_bounds__(kThreads) k_gather_copy(const __grid_constant__ Pieces pc, int64_t nvec,
                                                          uint4* __restrict__ out,
                                                          const __grid_constant__ SyncArgs sy) {
  if (!sync_wait(sy)) return;
  const int lane = threadIdx.x & 31;
  const int64_t warp = global_warp();
  const int64_t nwarps = num_warps();
  const int64_t per = pc.len / 16;                 // uint4 per piece
  const int64_t tpp = (per + 32 * U - 1) / (32 * U);   // tiles per piece
  (void)nvec;
  for (int64_t tile = warp; tile < tpp * pc.n; tile += nwarps) {
    const int j = static_cast<int>(tile % pc.n);
    const int64_t vb = (tile / pc.n) * (32 * U);   // first uint4 of the tile within piece j
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = vb + u * 32 + lane;
      if (q < per) r[u] = HZ_PEER_LD(reinterpret_cast<const uint4*>(pc.c[j]) + q);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = vb + u * 32 + lane;
      if (q < per) out[j * per + q] = r[u];
    }
  }
  sync_signal(sy);
}

template <typename TO, int U>
cudaError_t adamw_u(const float* g, float* th, float* m, float* v, void* out, int64_t n, const AdamW& hp,
                    cudaStream_t st, const SyncArgs& sy) {
  const int64_t n4 = n / 4;
  auto kern = k_adamw<TO, U>;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), (n4 + 32 * U - 1) / (32 * U));
  return launch_k(kern, grid, st, g, th, m, v, static_cast<TO*>(out), n4, hp, sy);
}

template <int GT, int U>
__global__ void __launch_bounds__(kThreads) k_sum_f32(const __grid_constant__ Pieces pc, int64_t n4,
                                                      float4* __restrict__ out, const __grid_constant__ SyncArgs sy) {
  if (!sync_wait(sy)) return;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
  const int64_t nth = static_cast<int64_t>(gridDim.x) * kThreads;
  const int g = GT > 0 ? GT : pc.n;
  for (int64_t base = tid; base < n4; base += nth * U) {
    float4 acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * nth;
      if (i < n4) acc[u] = HZ_PEER_LD(reinterpret_cast<const float4*>(pc.c[0]) + i);
    }
    for (int j = 1; j < g; ++j) {
      float4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = base + u * nth;
        if (i < n4) x[u] = HZ_PEER_LD(reinterpret_cast<const float4*>(pc.c[j]) + i);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc[u].x = __fadd_rn(acc[u].x, x[u].x);
        acc[u].y = __fadd_rn(acc[u].y, x[u].y);
        acc[u].z = __fadd_rn(acc[u].z, x[u].z);
        acc[u].w = __fadd_rn(acc[u].w, x[u].w);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * nth;
      if (i < n4) out[i] = acc[u];
    }
  }
  sync_signal(sy);
}

template <int GT>
cudaError_t sum_t(const Pieces& pc, int64_t n, float* out, cudaStream_t st, const SyncArgs& sy) {
  constexpr int U = 2;
  const int64_t n4 = n / 4;
  auto kern = k_sum_f32<GT, U>;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), (n4 + 32 * U - 1) / (32 * U));
  return launch_k(kern, grid, st, pc, n4, reinterpret_cast<float4*>(out), sy);
}

template <typename TO>
cudaError_t adamw_t(const float* g, float* th, float* m, float* v, void* out, int64_t n, const AdamW& hp,
                    cudaStream_t st, const SyncArgs& sy) {
  // HZ_TUNE adamw_u: float4 groups in flight per thread.  1 (40 registers, 6 CTAs per SM)
  // measured 5.9 TB/s on the 1.3B step tail vs 4.8 (u=2, 76 registers) and 4.0 (u=4)
  switch (tune_param("adamw_u", 1)) {
    case 2: return adamw_u<TO, 2>(g, th, m, v, out, n, hp, st, sy);
    case 4: return adamw_u<TO, 4>(g, th, m, v, out, n, hp, st, sy);
    default: return adamw_u<TO, 1>(g, th, m, v, out, n, hp, st, sy);
  }
}

}  // namespace

cudaError_t launch_adamw(const float* g, float* th, float* m, float* v, void* out, hz_dtype out_dt, int64_t n,
                         const AdamW& hp, cudaStream_t st, const SyncArgs* sync) {
  const SyncArgs sy = sync ? *sync : SyncArgs{};
  if (n == 0 && !sync) return cudaSuccess;
  switch (out_dt) {
    case HZ_F32: return adamw_t<float>(g, th, m, v, out, n, hp, st, sy);
    case HZ_BF16: return adamw_t<__nv_bfloat16>(g, th, m, v, out, n, hp, st, sy);
    case HZ_F16: return adamw_t<__half>(g, th, m, v, out, n, hp, st, sy);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_sum_f32(const Pieces& pc, int64_t n, float* out, cudaStream_t st, const SyncArgs* sync) {
  const SyncArgs sy = sync ? *sync : SyncArgs{};
  if (n == 0 && !sync) return cudaSuccess;
  switch (pc.n) {
    case 1: return sum_t<1>(pc, n, out, st, sy);
    case 2: return sum_t<2>(pc, n, out, st, sy);
    case 4: return sum_t<4>(pc, n, out, st, sy);
    case 8: return sum_t<8>(pc, n, out, st, sy);
    default: return sum_t<0>(pc, n, out, st, sy);
  }
}

cudaError_t launch_gather_copy(const Pieces& pc, void* out, cudaStream_t st, const SyncArgs* sync) {
  const SyncArgs sy = sync ? *sync : SyncArgs{};
  constexpr int U = 4;
  const int64_t nvec = pc.n * (pc.len / 16);
  auto kern = k_gather_copy<U>;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), (nvec + 32 * U - 1) / (32 * U));
  return launch_k(kern, grid, st, pc, nvec, static_cast<uint4*>(out), sy);
}

}  // namespace hz

// ---------------------------------------------------------------- NVLink probe
// hz_nvlink_probe: how fast this GPU's SMs pull a peer's memory with the same load
// path the fused gather / reduce kernels use (16-byte HZ_PEER_LD loads, U in flight
// per thread, grid = SMs x resident CTAs).  The XOR of what a CTA read goes to
// sink[blockIdx.x] so the loads cannot be elided.
namespace hz {
namespace {
template <int U>
__global__ void __launch_bounds__(dev::kThreads) k_peer_read(const uint4* __restrict__ src, int64_t n16,
                                                            unsigned* __restrict__ sink) {
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * dev::kThreads + threadIdx.x;
  const int64_t nth = static_cast<int64_t>(gridDim.x) * dev::kThreads;
  unsigned acc = 0;
  for (int64_t base = tid; base < n16; base += nth * U) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * nth;
      r[u] = i < n16 ? HZ_PEER_LD(src + i) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= r[u].x ^ r[u].y ^ r[u].z ^ r[u].w;
  }
  acc = __reduce_xor_sync(0xffffffffu, acc);
  if ((threadIdx.x & 31) == 0) atomicXor(sink + blockIdx.x, acc);
}
}  // namespace

cudaError_t launch_peer_read(const void* src, int64_t bytes, unsigned* sink, cudaStream_t st) {
  constexpr int U = 8;
  auto kern = k_peer_read<U>;
  const int64_t n16 = bytes / 16;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), (n16 + 32 * U - 1) / (32 * U));
  return launch_k(kern, grid, st, static_cast<const uint4*>(src), n16, sink);
}
}  // namespace hz
