// Fused codec + NVLink collective kernels (P2P transport, B = 256): one launch per
// collective call in which production (quantize) and consumption (peer loads +
// dequantize / reduce) overlap chunk by chunk.
//
//   k_ag_fused   qwZ forward all-gather (A2 + A3 + A5): quantize the
//                own primary into the peer-readable buffer, publish per-chunk
//                ready flags to every member, and dequantize every member's
//                chunks (read straight from its pool over NVLink) into the layer.
//   k_rs_fused   first qgZ level (A7 + A8 + A9): quantize the own
//                gradient chunk by chunk (chunks for all destinations interleaved),
//                publish each chunk's flag to its destination member, and reduce
//                the members' chunks destined to this rank (ascending digit, fp32,
//                no FMA) into the fp32 shard or the next level's requantized buffer.
//
// STATUS: experimental, off by default (HZ_TUNE fused=1).  Measured on 2 B200s at
// GPT-1.3B layer size these are slower than the two-kernel P2P path (74 vs 59 µs
// for the forward gather, 83 vs 49 µs for the qgZ level): a work item is one
// 32K-element chunk processed by one CTA, and that serialisation costs more than
// the overlap gains.  Kept (and parity-tested with fused=1) for a finer-grained
// interleaved design.
//
// Work distribution: persistent CTAs take work items from a global counter —
// first every production item, then the consumption items (remote pieces before
// the own one).  A consumption item waits (thread 0, ld.acquire.sys) for the
// chunk flags it needs; every item a CTA waits for has already been taken by a
// running CTA (here or on the producing peer), so the waits always make progress
// and no co-residency of the whole grid is required.  The whole call is one phase
// of the P2P protocol (codec.cuh): prologue waits until every rank is done with the
// previous phase; the last CTA publishes done (and, with requantization, ready for
// the next level).  Chunk flags hold the phase number (relative to the graph epoch).
#include "codec.cuh"

namespace hz {
namespace {

using namespace dev;
constexpr int kB = 256;                 // block size of the fused kernels
constexpr int kWarps = kThreads / 32;

struct FusedAG {
  const void* x;                        // own primary, plen elements
  uint8_t* qc;                          // own quantized primary (peer-readable)
  float* qs;
  const uint8_t* pc[kMaxWorld];         // member j's quantized primary (piece j)
  const float* ps[kMaxWorld];
  int D, me;
  int64_t plen, C;
  int nch;
  unsigned long long* flags;            // local [kMaxWorld][kMaxChunks]: flag[j][c] set by member j
  unsigned long long* flags_remote[kMaxWorld];   // &flag[me][0] in member j's pool
  unsigned long long* work;             // [0] work counter, [1] arrival counter (local)
  void* y;                              // the layer, D * plen elements
  unsigned long long phase;             // relative to *epoch
  const unsigned long long* epoch;
};

struct FusedRS {
  const void* x;                        // own input over range_{l-1}: g * cl elements
  uint8_t* qc;                          // own send buffer (peer-readable)
  float* qs;
  const uint8_t* mc[kMaxG];             // member j's send buffer at the chunk destined to me
  const float* ms[kMaxG];
  int g, d, bits_out, acc;
  int64_t cl, C;
  int ncl;                              // chunks per destination
  unsigned long long* flags;            // local [kMaxG][kMaxChunks]: flag[j][c] set by member j
  unsigned long long* flags_remote[kMaxG];       // &flag[d][0] in member j's pool
  unsigned long long* work;
  float* of;                            // fp32 output (bits_out == 0)
  uint8_t* oc;                          // requantized output (bits_out 4 / 8)
  float* os;
  unsigned long long phase;
  const unsigned long long* epoch;
};

__device__ __forceinline__ long long grab(unsigned long long* work) {
  __shared__ long long s_item;
  if (threadIdx.x == 0) s_item = static_cast<long long>(atomicAdd(work, 1ull));
  __syncthreads();
  const long long it = s_item;
  __syncthreads();
  return it;
}

__device__ __forceinline__ void wait_flag(const unsigned long long* f, unsigned long long target) {
  if (threadIdx.x == 0) {
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(f) < target)
      if (globaltimer() - t0 > 20000000000ull) __trap();
  }
  __syncthreads();
}

__device__ __forceinline__ void publish(unsigned long long* const* dst, int n, int64_t idx,
                                        unsigned long long v) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    for (int j = 0; j < n; ++j) st_relaxed_sys(dst[j] + idx, v);
  }
}

__device__ __forceinline__ void finish(unsigned long long* work) {
  // the last CTA resets the work counter for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(work + 1, 1ull) == gridDim.x - 1ull) {
      work[0] = 0ull;
      work[1] = 0ull;
      __threadfence();
    }
  }
}

// Quantize elements [e0, e0 + n) of x (n a multiple of 1024) into codes / scales at
// the same offsets: warp iterations of 4 blocks, one division per block.
template <typename T, int BITS>
__device__ __forceinline__ void cta_quantize(const T* __restrict__ x, int64_t e0, int64_t n,
                                             uint8_t* __restrict__ codes, float* __restrict__ scales) {
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  for (int64_t it = w; it < n / (kB * U); it += kWarps) {
    const int64_t blk0 = (e0 / kB) + it * U;
    In8<T> raw[U][1];
#pragma unroll
    for (int u = 0; u < U; ++u) raw[u][0].load(x + (blk0 + u) * kB + lane * 8);
    float v[U][1][8];
    float am[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      raw[u][0].get(v[u][0]);
      float m = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) m = fmaxf(m, fabsf(v[u][0][i]));
      am[u] = group_max<32>(m);
    }
    quantize_store<kB, BITS, U>(v, am, blk0, lane, codes, scales);
  }
}

// Dequantize n elements (multiple of 8) from codes / scales (maybe peer memory) to y.
template <int BITS, typename TO>
__device__ __forceinline__ void cta_dequantize(const uint8_t* __restrict__ codes, const float* __restrict__ scales,
                                               int64_t n, TO* __restrict__ y) {
  constexpr int U = 4;
  const int64_t nunits = n / 8;
  for (int64_t base = threadIdx.x; base < nunits; base += kThreads * U) {
    Codes8<BITS> raw[U];
    float sc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t unit = base + u * kThreads;
      if (unit < nunits) {
        raw[u].load(codes + unit * BITS);
        sc[u] = __ldg(scales + (unit * 8) / kB);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t unit = base + u * kThreads;
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

template <typename T, int BITS, typename TO>
__global__ void __launch_bounds__(kThreads) k_ag_fused(const __grid_constant__ FusedAG a,
                                                       const __grid_constant__ SyncArgs sy) {
  sync_wait(sy);   // every rank is done with the previous phase: our buffer is free
  const unsigned long long target = a.phase + (a.epoch ? *a.epoch : 0ull);
  const long long nprod = a.nch;
  const long long nremote = static_cast<long long>(a.D - 1) * a.nch;
  const long long ntotal = nprod + nremote + a.nch;
  for (;;) {
    const long long item = grab(a.work);
    if (item >= ntotal) break;
    if (item < nprod) {                                   // produce own chunk
      const int64_t e0 = item * a.C;
      const int64_t n = min(a.C, a.plen - e0);
      cta_quantize<T, BITS>(static_cast<const T*>(a.x), e0, n, a.qc, a.qs);
      publish(a.flags_remote, a.D, item, target);
    } else {                                              // consume a member's chunk
      long long k = item - nprod;
      int piece;
      int64_t c;
      if (k < nremote) {
        const int jj = static_cast<int>(k / a.nch);
        piece = jj < a.me ? jj : jj + 1;
        c = k % a.nch;
      } else {
        piece = a.me;
        c = k - nremote;
      }
      wait_flag(a.flags + static_cast<int64_t>(piece) * kMaxChunks + c, target);
      const int64_t e0 = c * a.C;
      const int64_t n = min(a.C, a.plen - e0);
      cta_dequantize<BITS, TO>(a.pc[piece] + e0 * BITS / 8, a.ps[piece] + e0 / kB, n,
                               static_cast<TO*>(a.y) + piece * a.plen + e0);
    }
  }
  finish(a.work);
  sync_signal(sy);   // done(phase)
}

// ------------------------------------------------------------------------ RS
// Reduce n elements (multiple of 256) of GT inputs into fp32 (staged, coalesced).
template <int BIN, int GT>
__device__ __forceinline__ void cta_reduce_f32(const FusedRS& a, int64_t off, int64_t n, float4* stage) {
  constexpr int E = 64 / BIN;
  constexpr int G = E / 4;
  constexpr int U = 2;                                  // warp chunks in flight per warp
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int64_t nunits = n / E;                         // a multiple of 32 * U * kWarps
  float4* st = stage + w * 32 * G;
  for (int64_t base0 = w * 32 * U; base0 < nunits; base0 += kThreads * U) {
  uint2 rawu[U][GT];
  float scu[U][GT];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int p = 0; p < GT; ++p) {
      const int64_t unit = base0 + u * 32 + lane;
      rawu[u][p] = __ldg(reinterpret_cast<const uint2*>(a.mc[p] + (off / E + unit) * 8));
      scu[u][p] = __ldg(a.ms[p] + (off + unit * E) / kB);
    }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t base = base0 + u * 32;
    float acc[E];
    const uint2 (&raw)[GT] = rawu[u];
    const float (&sc)[GT] = scu[u];
#pragma unroll
    for (int p = 0; p < GT; ++p) {
      float c[E];
      if constexpr (BIN == 8) {
        Codes8<8> cc;
        cc.r = raw[p];
        cc.decode(c);
      } else {
        Codes8<4> lo, hi;
        lo.r = raw[p].x;
        hi.r = raw[p].y;
        float t0[8], t1[8];
        lo.decode(t0);
        hi.decode(t1);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          c[i] = t0[i];
          c[8 + i] = t1[i];
        }
      }
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const float xh = __fmul_rn(c[i], sc[p]);
        acc[i] = p == 0 ? xh : __fadd_rn(acc[i], xh);
      }
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const int gi = lane * G + j;
      st[gi ^ ((gi >> 3) & (G - 1))] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const int gi = k * 32 + lane;
      float4 o = st[gi ^ ((gi >> 3) & (G - 1))];
      float4* dst = reinterpret_cast<float4*>(a.of + off) + base * G + gi;
      if (a.acc) {
        const float4 old = *dst;
        o.x = __fadd_rn(old.x, o.x);
        o.y = __fadd_rn(old.y, o.y);
        o.z = __fadd_rn(old.z, o.z);
        o.w = __fadd_rn(old.w, o.w);
      }
      *dst = o;
    }
    __syncwarp();
  }
  }
}

// Reduce + requantize n elements (multiple of 1024) of GT inputs into oc / os at off.
template <int BIN, int BOUT, int GT>
__device__ __forceinline__ void cta_reduce_requant(const FusedRS& a, int64_t off, int64_t n) {
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  for (int64_t it = w; it < n / (kB * U); it += kWarps) {
    const int64_t blk0 = off / kB + it * U;
    float v[U][1][8];
    float am[U];
    Codes8<BIN> raw[U][GT];
    float sc[U][GT];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int p = 0; p < GT; ++p) {
        raw[u][p].load(a.mc[p] + ((blk0 + u) * kB + lane * 8) * BIN / 8);
        sc[u][p] = __ldg(a.ms[p] + blk0 + u);
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float c[8];
#pragma unroll
      for (int p = 0; p < GT; ++p) {
        raw[u][p].decode(c);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float xh = __fmul_rn(c[i], sc[u][p]);
          v[u][0][i] = p == 0 ? xh : __fadd_rn(v[u][0][i], xh);
        }
      }
      float m = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) m = fmaxf(m, fabsf(v[u][0][i]));
      am[u] = group_max<32>(m);
    }
    quantize_store<kB, BOUT, U>(v, am, blk0, lane, a.oc, a.os);
  }
}

template <typename T, int BIN, int BOUT, int GT>
__global__ void __launch_bounds__(kThreads) k_rs_fused(const __grid_constant__ FusedRS a,
                                                       const __grid_constant__ SyncArgs sy) {
  __shared__ float4 stage[BOUT == 0 ? kThreads / 32 * 32 * (16 / BIN) : 1];
  sync_wait(sy);
  const unsigned long long target = a.phase + (a.epoch ? *a.epoch : 0ull);
  const long long nprod = static_cast<long long>(a.g) * a.ncl;
  const long long ntotal = nprod + a.ncl;
  for (;;) {
    const long long item = grab(a.work);
    if (item >= ntotal) break;
    if (item < nprod) {   // produce: destinations interleaved so every member's chunks come early
      const int dest = static_cast<int>(item % a.g);
      const int64_t c = item / a.g;
      const int64_t e0 = dest * a.cl + c * a.C;
      const int64_t n = min(a.C, a.cl - c * a.C);
      cta_quantize<T, BIN>(static_cast<const T*>(a.x), e0, n, a.qc, a.qs);
      publish(a.flags_remote + dest, 1, c, target);
    } else {
      const int64_t c = item - nprod;
      for (int j = 0; j < GT; ++j) wait_flag(a.flags + static_cast<int64_t>(j) * kMaxChunks + c, target);
      const int64_t off = c * a.C;
      const int64_t n = min(a.C, a.cl - off);
      if constexpr (BOUT == 0) cta_reduce_f32<BIN, GT>(a, off, n, stage);
      else cta_reduce_requant<BIN, BOUT, GT>(a, off, n);
    }
  }
  finish(a.work);
  sync_signal(sy);
}

int64_t fused_grid(const void* kernel, int64_t items) {
  return grid_for(kernel, items * kWarps);   // at most one CTA per work item
}

template <typename T, int BITS, typename TO>
cudaError_t ag_t(const FusedAG& a, cudaStream_t st, const SyncArgs& sy) {
  auto kern = k_ag_fused<T, BITS, TO>;
  const int64_t grid = fused_grid(reinterpret_cast<const void*>(kern), static_cast<int64_t>(a.D + 1) * a.nch);
  kern<<<static_cast<unsigned>(grid), kThreads, 0, st>>>(a, sy);
  return cudaGetLastError();
}

template <typename T, int BITS>
cudaError_t ag_o(const FusedAG& a, hz_dtype out_dt, cudaStream_t st, const SyncArgs& sy) {
  switch (out_dt) {
    case HZ_BF16: return ag_t<T, BITS, __nv_bfloat16>(a, st, sy);
    case HZ_F16: return ag_t<T, BITS, __half>(a, st, sy);
    case HZ_F32: return ag_t<T, BITS, float>(a, st, sy);
  }
  return cudaErrorInvalidValue;
}

template <typename T, int BIN, int BOUT, int GT>
cudaError_t rs_t(const FusedRS& a, cudaStream_t st, const SyncArgs& sy) {
  auto kern = k_rs_fused<T, BIN, BOUT, GT>;
  const int64_t grid = fused_grid(reinterpret_cast<const void*>(kern), static_cast<int64_t>(a.g + 1) * a.ncl);
  kern<<<static_cast<unsigned>(grid), kThreads, 0, st>>>(a, sy);
  return cudaGetLastError();
}

template <typename T, int BIN, int BOUT>
cudaError_t rs_g(const FusedRS& a, cudaStream_t st, const SyncArgs& sy) {
  switch (a.g) {
    case 2: return rs_t<T, BIN, BOUT, 2>(a, st, sy);
    case 4: return rs_t<T, BIN, BOUT, 4>(a, st, sy);
    case 8: return rs_t<T, BIN, BOUT, 8>(a, st, sy);
  }
  return cudaErrorInvalidValue;
}

template <typename T, int BIN>
cudaError_t rs_o(const FusedRS& a, cudaStream_t st, const SyncArgs& sy) {
  switch (a.bits_out) {
    case 0: return rs_g<T, BIN, 0>(a, st, sy);
    case 4: return rs_g<T, BIN, 4>(a, st, sy);
    case 8: return rs_g<T, BIN, 8>(a, st, sy);
  }
  return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t rs_b(const FusedRS& a, int bits_in, cudaStream_t st, const SyncArgs& sy) {
  return bits_in == 8 ? rs_o<T, 8>(a, st, sy) : rs_o<T, 4>(a, st, sy);
}

}  // namespace

bool fused_rs_supported(int g) { return g == 2 || g == 4 || g == 8; }

cudaError_t launch_ag_fused(const FusedAGArgs& h, cudaStream_t st, const SyncArgs& sy) {
  FusedAG a{};
  a.x = h.x;
  a.qc = h.qc;
  a.qs = h.qs;
  for (int j = 0; j < h.D; ++j) {
    a.pc[j] = h.pc[j];
    a.ps[j] = h.ps[j];
    a.flags_remote[j] = h.flags_remote[j];
  }
  a.D = h.D;
  a.me = h.me;
  a.plen = h.plen;
  a.C = h.C;
  a.nch = h.nch;
  a.flags = h.flags;
  a.work = h.work;
  a.y = h.y;
  a.phase = h.phase;
  a.epoch = h.epoch;
  if (h.bits == 8) {
    switch (h.dt) {
      case HZ_BF16: return ag_o<__nv_bfloat16, 8>(a, h.out_dt, st, sy);
      case HZ_F16: return ag_o<__half, 8>(a, h.out_dt, st, sy);
      case HZ_F32: return ag_o<float, 8>(a, h.out_dt, st, sy);
    }
  } else {
    switch (h.dt) {
      case HZ_BF16: return ag_o<__nv_bfloat16, 4>(a, h.out_dt, st, sy);
      case HZ_F16: return ag_o<__half, 4>(a, h.out_dt, st, sy);
      case HZ_F32: return ag_o<float, 4>(a, h.out_dt, st, sy);
    }
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_rs_fused(const FusedRSArgs& h, cudaStream_t st, const SyncArgs& sy) {
  FusedRS a{};
  a.x = h.x;
  a.qc = h.qc;
  a.qs = h.qs;
  for (int j = 0; j < h.g; ++j) {
    a.mc[j] = h.mc[j];
    a.ms[j] = h.ms[j];
    a.flags_remote[j] = h.flags_remote[j];
  }
  a.g = h.g;
  a.d = h.d;
  a.bits_out = h.bits_out;
  a.acc = h.acc;
  a.cl = h.cl;
  a.C = h.C;
  a.ncl = h.ncl;
  a.flags = h.flags;
  a.work = h.work;
  a.of = h.of;
  a.oc = h.oc;
  a.os = h.os;
  a.phase = h.phase;
  a.epoch = h.epoch;
  switch (h.dt) {
    case HZ_BF16: return rs_b<__nv_bfloat16>(a, h.bits_in, st, sy);
    case HZ_F16: return rs_b<__half>(a, h.bits_in, st, sy);
    case HZ_F32: return rs_b<float>(a, h.bits_in, st, sy);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hz
