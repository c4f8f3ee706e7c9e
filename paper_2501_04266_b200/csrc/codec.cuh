// Device helpers shared by the sm_100a codec kernels (k_quantize.cu,
// k_dequantize.cu, k_reduce.cu).  Internal header.
//
// Exactness (oracle readings R1-R5): every operation below
// rounds exactly like the oracle's fp32 NumPy code.
//   * bf16/fp16 -> fp32 widening is exact.
//   * scale = __fdiv_rn(am, qmax), inv = __fdiv_rn(qmax, am) (IEEE division).
//   * code = rne(fl(x*inv)) is computed as fl(fl(x*inv) + 1.5*2^23): for
//     |t| <= 2^22 the sum lands in [2^23, 2^24) where the fp32 spacing is 1, so
//     round-to-nearest-even of the sum IS rint(t), and the low bits of the sum's
//     bit pattern are rint(t) in two's complement.  This replaces F2I (a
//     quarter-rate conversion) by one full-rate FADD.  The two roundings are
//     kept separate (--fmad=false, explicit __fmul_rn/__fadd_rn): a fused FMA
//     would round x*inv + M once and could differ next to a tie.
//   * no clamp is needed: |x| <= am and inv <= (qmax/am)(1 + 2^-24), so
//     |fl(x*inv)| <= qmax*(1 + 2^-23) < qmax + 1/2 and rint stays in
//     [-qmax, qmax] (the oracle's clamp is provably inactive).
//   * code -> float uses the same trick backwards: a byte / nibble placed in the
//     low bits of 0x4B400000 reads as 1.5*2^23 + k; subtracting the exact bias
//     gives the integer code exactly (replaces I2F).
//   * x_hat = __fmul_rn(code, scale); sums use __fadd_rn in ascending input order.
// Loads: inputs only this GPU writes (the primary, the gradient) use the read-only
// path (__ldg); codes and scales, which may be a peer's IPC-mapped memory written by
// that peer while this kernel's grid is alive, use coherent L2 loads (__ldcg,
// ld.global.cg: no L1 allocation), ordered after the phase wait (codec.cuh bottom).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <utility>

#include "hz_internal.h"

// load of codes / scales that may be peer memory (see the header comment)
#ifndef HZ_PEER_LD
#define HZ_PEER_LD __ldcg
#endif

namespace hz {
namespace dev {

constexpr unsigned kFull = 0xffffffffu;
constexpr float kTiny = 0x1p-100f;        // R3: am < 2^-100 -> scale 0, codes 0
constexpr float kMagic = 12582912.0f;     // 1.5 * 2^23, bit pattern 0x4B400000
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
  __device__ __forceinline__ void load_shared(const float* p) {   // tile engine: a staged tile
    r[0] = reinterpret_cast<const uint4*>(p)[0];
    r[1] = reinterpret_cast<const uint4*>(p)[1];
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
  __device__ __forceinline__ void load_shared(const __nv_bfloat16* p) { r = *reinterpret_cast<const uint4*>(p); }
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
  __device__ __forceinline__ void load_shared(const __half* p) { r = *reinterpret_cast<const uint4*>(p); }
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

// ------------------------------------------------------------------ codes
// byte i of x (bias 128 already applied) -> 1.5*2^23 + byte
__device__ __forceinline__ float byte_as_magic(unsigned x, int i) {
  return __uint_as_float(__byte_perm(x, 0x4B400000u, 0x7650u + i));
}

// 8 int8 codes (8 bytes)
template <int BITS>
struct Codes8;

template <>
struct Codes8<8> {
  uint2 r;
  __device__ __forceinline__ void load(const uint8_t* p) { r = HZ_PEER_LD(reinterpret_cast<const uint2*>(p)); }
  __device__ __forceinline__ void load_shared(const void* p) { r = *reinterpret_cast<const uint2*>(p); }
  __device__ __forceinline__ void store(uint8_t* p) const { *reinterpret_cast<uint2*>(p) = r; }
  __device__ __forceinline__ void zero() { r = make_uint2(0u, 0u); }
  // exact float value of each code
  __device__ __forceinline__ void decode(float (&c)[8]) const {
    const unsigned x = r.x ^ 0x80808080u, y = r.y ^ 0x80808080u;   // two's complement -> +128 bias
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      c[i] = __fsub_rn(byte_as_magic(x, i), kMagic + 128.f);
      c[4 + i] = __fsub_rn(byte_as_magic(y, i), kMagic + 128.f);
    }
  }
  // b[i] = bit pattern of fl(t_i + 1.5*2^23): its low byte is code i
  __device__ __forceinline__ void set(const unsigned (&b)[8]) {
    r.x = __byte_perm(__byte_perm(b[0], b[1], 0x0040u), __byte_perm(b[2], b[3], 0x0040u), 0x5410u);
    r.y = __byte_perm(__byte_perm(b[4], b[5], 0x0040u), __byte_perm(b[6], b[7], 0x0040u), 0x5410u);
  }
};

// 8 int4 codes (4 bytes), even element in the low nibble (R4)
template <>
struct Codes8<4> {
  unsigned r;
  __device__ __forceinline__ void load(const uint8_t* p) { r = HZ_PEER_LD(reinterpret_cast<const unsigned*>(p)); }
  __device__ __forceinline__ void load_shared(const void* p) { r = *reinterpret_cast<const unsigned*>(p); }
  __device__ __forceinline__ void store(uint8_t* p) const { *reinterpret_cast<unsigned*>(p) = r; }
  __device__ __forceinline__ void zero() { r = 0u; }
  __device__ __forceinline__ void decode(float (&c)[8]) const {
    // nibble ^ 8 = code + 8 in [1, 15]; even / odd nibbles spread to bytes, then each
    // byte is placed in the mantissa of 1.5*2^23 and the bias M + 8 removed.
    const unsigned x = r ^ 0x88888888u;
    const unsigned ev = x & 0x0F0F0F0Fu;           // codes 0, 2, 4, 6
    const unsigned od = (x >> 4) & 0x0F0F0F0Fu;    // codes 1, 3, 5, 7
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      c[2 * i] = __fsub_rn(byte_as_magic(ev, i), kMagic + 8.f);
      c[2 * i + 1] = __fsub_rn(byte_as_magic(od, i), kMagic + 8.f);
    }
  }
  __device__ __forceinline__ void set(const unsigned (&b)[8]) {
    unsigned n[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) n[i] = (b[2 * i] & 0xFu) | ((b[2 * i + 1] << 4) & 0xF0u);
    r = __byte_perm(__byte_perm(n[0], n[1], 0x0040u), __byte_perm(n[2], n[3], 0x0040u), 0x5410u);
  }
};

// 4 codes (elementwise kernels with 4-element units)
template <int BITS>
struct Codes4;

template <>
struct Codes4<8> {
  unsigned r;
  __device__ __forceinline__ void load(const uint8_t* p) { r = HZ_PEER_LD(reinterpret_cast<const unsigned*>(p)); }
  __device__ __forceinline__ void load_shared(const void* p) { r = *reinterpret_cast<const unsigned*>(p); }
  __device__ __forceinline__ void decode(float (&c)[4]) const {
    const unsigned x = r ^ 0x80808080u;
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i] = __fsub_rn(byte_as_magic(x, i), kMagic + 128.f);
  }
};

template <>
struct Codes4<4> {
  unsigned short r;
  __device__ __forceinline__ void load(const uint8_t* p) {
    r = HZ_PEER_LD(reinterpret_cast<const unsigned short*>(p));
  }
  __device__ __forceinline__ void load_shared(const void* p) { r = *reinterpret_cast<const unsigned short*>(p); }
  __device__ __forceinline__ void decode(float (&c)[4]) const {
    const unsigned x = static_cast<unsigned>(r) ^ 0x8888u;   // nibble ^ 8 = code + 8
    const unsigned ev = x & 0x0F0Fu;
    const unsigned od = (x >> 4) & 0x0F0Fu;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      c[2 * i] = __fsub_rn(byte_as_magic(ev, i), kMagic + 8.f);
      c[2 * i + 1] = __fsub_rn(byte_as_magic(od, i), kMagic + 8.f);
    }
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

// bit pattern of fl(fl(v*inv) + 1.5*2^23); low bits = rne(fl(v*inv)) (see header)
__device__ __forceinline__ unsigned qbits(float v, float inv) {
  return __float_as_uint(__fadd_rn(__fmul_rn(v, inv), kMagic));
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
    unsigned w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);   // RNE
      w[i] = *reinterpret_cast<unsigned*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};

template <>
struct Out8<__half> {
  __device__ __forceinline__ static void store(__half* p, const float (&v)[8]) {
    unsigned w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);              // RNE
      w[i] = *reinterpret_cast<unsigned*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};

// Quantize-and-store epilogue shared by k_quantize and k_reduce_requant for one
// warp iteration of U full warp steps (NB = U * BPW consecutive blocks starting
// at blk0; no bounds checks).  am[u] must already be the group-reduced absmax of
// this lane's block in step u.  The scale / inv divisions run once per block:
// lane k (< NB) divides for block k, then inv is broadcast back by shuffle, and
// lanes 0..NB-1 store the NB consecutive scales in one coalesced store.
//
// Emit (optional) receives the dequantized value x_hat = fl(code * scale) of the
// lane's 8 elements starting at global element e0, warp-uniformly: the fused
// quantize -> dequantize of a level without exchange (group size 1).
struct NoEmit {
  static constexpr bool on = false;
  __device__ __forceinline__ void operator()(int64_t, int, const float (&)[8]) const {}
};

template <int B, int BITS, int U, class Emit = NoEmit>
__device__ __forceinline__ void quantize_store(const float (&v)[U][Geo<B>::NSUB][8], const float (&am)[U],
                                               int64_t blk0, int lane, uint8_t* __restrict__ codes,
                                               float* __restrict__ scales, const Emit& emit = Emit{}) {
  using G = Geo<B>;
  constexpr int NB = U * G::BPW;
  static_assert(NB <= 32, "one block per lane at most");
  const int lb = lane / G::LPB;
  const int ll = lane % G::LPB;
  float mine = 0.f;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const float t = __shfl_sync(kFull, am[u], (lane % G::BPW) * G::LPB);
    if (lane / G::BPW == u) mine = t;
  }
  float scale, inv;
  quant_params<BITS>(mine, scale, inv);
  // codes == nullptr (round trip of a one-member level): no code / scale stores
  if (codes && lane < NB) scales[blk0 + lane] = scale;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const float iv = __shfl_sync(kFull, inv, u * G::BPW + lb);
    const float sc = Emit::on ? __shfl_sync(kFull, scale, u * G::BPW + lb) : 0.f;
    const int64_t blk = blk0 + u * G::BPW + lb;
#pragma unroll
    for (int k = 0; k < G::NSUB; ++k) {
      unsigned b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) b[i] = qbits(v[u][k][i], iv);
      if (codes) {
        Codes8<BITS> out;
        out.set(b);
        out.store(codes + (blk * B + k * G::SUBSTRIDE + ll * 8) * BITS / 8);
      }
      if constexpr (Emit::on) {
        float xh[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) xh[i] = __fmul_rn(__fsub_rn(__uint_as_float(b[i]), kMagic), sc);
        emit(blk * B + k * G::SUBSTRIDE + ll * 8, lane, xh);
      }
    }
  }
}

// Emitters for the fused round trip.  16-bit outputs: one 16-byte store per lane
// (the lanes of a warp step own 256 consecutive elements).  fp32: staged through
// 1 KB of shared memory per warp (swizzled granules) so that each store, and the
// accumulate load, is one contiguous 512-byte span; A = fl(A + x_hat) when acc.
template <typename TO>
struct EmitOut {
  static constexpr bool on = true;
  TO* y;
  __device__ __forceinline__ void operator()(int64_t e0, int, const float (&xh)[8]) const {
    Out8<TO>::store(y + e0, xh);
  }
};

struct EmitF32 {
  static constexpr bool on = true;
  float* y;
  float4* stage;   // this warp's 64 granules
  int acc;
  __device__ __forceinline__ void operator()(int64_t e0, int lane, const float (&xh)[8]) const {
    const int64_t base = e0 - 8 * lane;   // first element of the warp step's 256
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int gi = lane * 2 + j;
      stage[gi ^ ((gi >> 3) & 1)] = make_float4(xh[4 * j], xh[4 * j + 1], xh[4 * j + 2], xh[4 * j + 3]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int gi = k * 32 + lane;
      float4 o = stage[gi ^ ((gi >> 3) & 1)];
      float4* dst = reinterpret_cast<float4*>(y + base) + gi;
      if (acc) {
        const float4 a = *dst;
        o.x = __fadd_rn(a.x, o.x);
        o.y = __fadd_rn(a.y, o.y);
        o.z = __fadd_rn(a.z, o.z);
        o.w = __fadd_rn(a.w, o.w);
      }
      *dst = o;
    }
    __syncwarp();
  }
};

// fp32 round trip without accumulate, stores by TMA: each warp step's 256 x_hat land in
// natural order in one of this warp's two 1 KB shared-memory buffers and lane 0 issues a
// cp.async.bulk shared -> global of the 1 KB span (the next-but-one step reuses a buffer
// after its bulk store has read it).  finish() waits for the warp's stores.  Values and
// rounding are EmitF32's.
struct EmitF32Bulk {
  static constexpr bool on = true;
  float* y;
  float4* stage;   // this warp's 2 x 64 granules
  mutable int buf;
  __device__ __forceinline__ void operator()(int64_t e0, int lane, const float (&xh)[8]) const {
    const int64_t base = e0 - 8 * lane;   // first element of the warp step's 256
    float4* st = stage + buf * 64;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    st[lane * 2] = make_float4(xh[0], xh[1], xh[2], xh[3]);
    st[lane * 2 + 1] = make_float4(xh[4], xh[5], xh[6], xh[7]);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 1024;" ::"l"(y + base),
                   "r"(static_cast<uint32_t>(__cvta_generic_to_shared(st)))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    buf ^= 1;
  }
  __device__ __forceinline__ void finish(int lane) const {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
};

// bf16 / fp16 round-trip output stored by TMA: as EmitF32Bulk with 512-byte spans (the
// 256 16-bit x_hat of a warp step), two buffers per warp.
template <typename TO>
struct EmitOutBulk {
  static constexpr bool on = true;
  TO* y;
  uint4* stage;   // this warp's 2 x 32 granules
  mutable int buf;
  __device__ __forceinline__ void operator()(int64_t e0, int lane, const float (&xh)[8]) const {
    const int64_t base = e0 - 8 * lane;
    uint4* st = stage + buf * 32;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    Out8<TO>::store(reinterpret_cast<TO*>(st) + lane * 8, xh);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(y + base),
                   "r"(static_cast<uint32_t>(__cvta_generic_to_shared(st)))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    buf ^= 1;
  }
  __device__ __forceinline__ void finish(int lane) const {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
};

__device__ __forceinline__ int64_t global_warp() {
  return (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
}
__device__ __forceinline__ int64_t num_warps() {
  return (static_cast<int64_t>(gridDim.x) * kThreads) >> 5;
}

}  // namespace dev

// host-side grid sizing (codec_util.cu): grid-stride kernels get
// min(ceil(warp_tasks / warps per CTA), SMs x resident CTAs of that kernel).
int64_t grid_for(const void* kernel, int64_t warp_tasks, int dyn_smem = 0);
int sm_count();   // SMs of the current device (cached)

// Every libhz kernel launch: kThreads per CTA, dynamic shared memory only for the link
// kernels (launch_k_smem; grid_for with the same dyn_smem sets the opt-in limit), and the
// programmatic-stream-serialization attribute when HZ_TUNE pdl=1 (PDL; off by
// default, see pdl_enabled) — the kernel's prologue (sync_wait) then orders it after
// the previous kernel on the stream; and the shared-memory carveout of the API call's
// CarveScope (hz_internal.h), when set.
bool pdl_enabled();
int launch_carve();
template <typename... KArgs, typename... Args>
cudaError_t launch_k_smem(void (*kern)(KArgs...), int64_t grid, int dyn_smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(dev::kThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(dyn_smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int carve = launch_carve();   // CarveScope of the API call (hz_internal.h)
  if (carve >= 0) {
    attr[1].id = cudaLaunchAttributePreferredSharedMemoryCarveout;
    attr[1].val.sharedMemCarveout = static_cast<unsigned>(carve);
    cfg.numAttrs = 2;
  }
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), int64_t grid, cudaStream_t st, Args&&... args) {
  return launch_k_smem(kern, grid, 0, st, std::forward<Args>(args)...);
}

}  // namespace hz

namespace hz {
// Launch-parameter overrides for tuning sweeps (tools/kbench.py --tune): the
// environment variable HZ_TUNE="name=value,..." is read once per process;
// unknown names fall back to the compiled defaults.  Product runs leave it unset.
int tune_param(const char* name, int dflt);
}  // namespace hz


// ======================================================================= P2P sync
// Cross-GPU phase synchronisation for the NVLink peer-memory transport (p2p.cpp).
// Every collective phase has a global number (the same on all ranks, which issue
// the same call sequence).  Flags live in each rank's IPC-mapped pool header:
// ready[q] / done[q] = the last phase rank q signalled to this rank (monotone).
// A kernel may
//   * wait (prologue, thread 0 of every CTA, ld.acquire.sys spin) until
//     ready[q] >= wait_ready for the ranks q of wr_mask (the members whose buffers
//     it reads) and done[q] >= wait_done for wd_mask (the ranks that read what it
//     overwrites) — level-local: no other rank is waited for;
//   * signal (epilogue, last CTA to finish, fence.acq_rel.sys + relaxed system-scope
//     stores) sig_ready to sr_mask and sig_done to sd_mask.
// A wait longer than timeout_ns, or a nonzero *abort (mapped host memory: set by
// another timed-out wait of this context, or by hz_abort on the host), aborts: the
// CTA returns without doing its work or signalling, *abort is set to 1, and the host
// reports HZ_ERR_ABORTED on the context's next call.  A dead or stalled peer
// therefore neither hangs the GPU nor leaves a sticky CUDA error.
namespace hz {
namespace dev {
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_volatile_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Returns false when the context is aborted (the whole CTA must return at once).
__device__ __forceinline__ bool sync_wait(const SyncArgs& s) {
  // Programmatic dependent launch (launch_k): let the next kernel on the stream be
  // launched now and wait here until the previous kernel has completed and its memory
  // is visible — the stream-order semantics minus the launch gap.  Both are no-ops
  // without the launch attribute.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (s.stamps && blockIdx.x == 0 && threadIdx.x == 0) s.stamps[0] = globaltimer();
  if (!(s.wr_mask | s.wd_mask)) {
    if (s.stamps && blockIdx.x == 0 && threadIdx.x == 0) s.stamps[1] = globaltimer();
    return true;
  }
  __shared__ int ok;
  if (threadIdx.x == 0) {
    const unsigned long long t0 = globaltimer();
    const unsigned long long e = s.epoch ? *s.epoch : 0ull;
    const unsigned long long wr = s.wait_ready + e, wd = s.wait_done + e;
    // the abort word lives in host memory: it is polled only once a wait has lasted
    // 1 ms, then every 100 us (hundreds of CTAs reading it on every entry would
    // serialise on PCIe)
    int good = 1;
    unsigned it = 0;
    unsigned long long next_poll = t0 + 1000000ull;
    for (int q = 0; q < kMaxWorld && good; ++q) {
      const bool r = (s.wr_mask >> q) & 1u, d = (s.wd_mask >> q) & 1u;
      while ((r && ld_acquire_sys(s.ready_local + q) < wr) || (d && ld_acquire_sys(s.done_local + q) < wd)) {
        if ((++it & 63u) == 0u) {
          const unsigned long long now = globaltimer();
          if (now >= next_poll) {
            next_poll = now + 100000ull;
            if (s.abort && ld_volatile_u32(s.abort) != 0u) {
              good = 0;
              break;
            }
          }
          if (now - t0 > s.timeout_ns) {
            if (s.abort) atomicExch(s.abort, 1u);
            good = 0;
            break;
          }
        }
      }
    }
    ok = good;
    if (s.stamps && blockIdx.x == 0) s.stamps[1] = globaltimer();
  }
  __syncthreads();
  return ok != 0;
}

// Kernel epilogue: trace stamp of the last CTA to finish (stamps[2], with its own
// arrival counter in stamps[4]) and, in P2P mode, the phase publication (stamps[3]).
__device__ __forceinline__ void sync_signal(const SyncArgs& s) {
  const bool sig = (s.sr_mask | s.sd_mask) != 0u;
  if (!sig && !s.stamps) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    // gpu-scope release per CTA (peers read this GPU's memory through its L2, the
    // point of coherence for gpu scope); the last CTA then publishes with a
    // system-scope acq_rel fence, cumulative over everything it has observed
    // (the arrival counter), followed by relaxed system-scope flag stores.
    __threadfence();
    if (s.stamps && atomicAdd(s.stamps + 4, 1ull) == gridDim.x - 1ull) {
      s.stamps[2] = globaltimer();
      s.stamps[4] = 0ull;   // graph replays reuse the slot
    }
    if (sig && atomicAdd(s.counter, 1u) == gridDim.x - 1) {
      *s.counter = 0u;
      const unsigned long long e = s.epoch ? *s.epoch : 0ull;
      const unsigned long long sr = s.sig_ready + e, sd = s.sig_done + e;
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      for (int q = 0; q < kMaxWorld; ++q) {
        if ((s.sr_mask >> q) & 1u) st_relaxed_sys(s.ready_remote[q], sr);
        if ((s.sd_mask >> q) & 1u) st_relaxed_sys(s.done_remote[q], sd);
      }
      if (s.stamps) s.stamps[3] = globaltimer();
    }
  }
}
}  // namespace dev
}  // namespace hz
