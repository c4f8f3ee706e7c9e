// Pipelined codec + NVLink collective kernels (P2P transport, B = 256): ONE launch
// per collective call in which production (quantize, HBM-bound) and consumption
// (peer loads + dequantize / reduce, NVLink-bound) run at the same time on
// different CTAs, chunk by chunk.
//
//   k_ag_pipe   qwZ forward all-gather (A2 + A3 + A5): producers
//               quantize the own primary into the peer-readable buffer chunk by
//               chunk and publish each chunk to every member; consumers dequantize
//               every member's chunk c (read straight from its pool over NVLink)
//               into the layer as soon as chunk c is published everywhere.
//   k_rs_pipe   first qgZ level (A7 + A8 + A9): producers quantize
//               the own gradient chunk c for every destination (int4/int8) and
//               publish it to its destination; consumers reduce the members' chunk
//               c destined here (ascending digit, fp32, no FMA) into the fp32 shard
//               or the next level's requantized send buffer.
//
// Roles: every CTA takes a ticket (atomicAdd on a local counter) at entry; the
// first Gp tickets are producers, the rest consumers.  A consumer only ever waits
// for chunks whose producers hold a ticket already (here and on every peer, since
// producers never wait), so the waits make progress however many CTAs are
// resident.  Within a role, CTAs stride over the chunk as one grid (virtual warp
// index = ticket * warps + warp), with the warp-level access pattern of the
// two-kernel path (k_quantize / k_dequantize / k_reduce).
//
// Chunk publication: a producer CTA finishing its part of chunk c fences (gpu
// scope) and increments the chunk's local arrival counter; the CTA completing the
// count issues fence.acq_rel.sys and stores the phase number into every member's
// flag for (this rank, c) — the cumulative last-CTA publication of the phase
// protocol in codec.cuh.  Flags hold the phase number relative to the graph epoch,
// so they never need resetting; the arrival counters and the ticket counter are
// reset by the last CTA of the launch.  The whole call is one phase: the prologue
// waits until every rank is done with the previous phase, the last CTA signals
// done(phase).
//
// Results are bit-identical to the two-kernel path (same per-block arithmetic,
// same summation order).  Selected with HZ_TUNE fused=1 (pf = producer share of
// the grid in %, pk = target chunks per call).
#include "codec.cuh"

namespace hz {
namespace {

using namespace dev;
constexpr int kB = 256;                 // block size of the pipelined kernels
constexpr int kWarps = kThreads / 32;
constexpr int kU = 4;                   // blocks (quantize) / 32-unit steps (consume) per warp item

struct FusedAG {
  const void* x;                        // own primary, plen elements
  uint8_t* qc;                          // own quantized primary (peer-readable)
  float* qs;
  const uint8_t* pc[kMaxWorld];         // member j's quantized primary (piece j)
  const float* ps[kMaxWorld];
  int D, me;
  int64_t plen, C;
  int nch;
  int gp;                               // producer CTAs
  unsigned long long* flags;            // local [kMaxWorld][kMaxChunks]: flag[j][c] set by member j
  unsigned long long* flags_remote[kMaxWorld];   // &flag[me][0] in member j's pool
  unsigned long long* work;             // [0] ticket counter, [1] exit counter (local)
  unsigned int* cnt;                    // [nch] producer arrivals per chunk (local)
  unsigned long long* dbg;              // optional timeline [c][4]: publish, first consumer start, last consumer end
  void* y;                              // the layer, D * plen elements
  unsigned long long phase;             // relative to *epoch
  const unsigned long long* epoch;
};

struct FusedRS {
  const void* x;                        // own input over range_{l-1}: g * cl elements
  uint8_t* qc;                          // own send buffer (peer-readable)
  float* qs;
  const uint8_t* mc[kMaxG];             // member j's send buffer at the slice destined to me
  const float* ms[kMaxG];
  int g, d, bits_out, acc;
  int64_t cl, C;
  int ncl;
  int gp;
  unsigned long long* flags;            // local [kMaxG][kMaxChunks]: flag[j][c] set by member j
  unsigned long long* flags_remote[kMaxG];       // &flag[d][0] in member j's pool
  unsigned long long* work;
  unsigned int* cnt;
  float* of;                            // fp32 output (bits_out == 0)
  uint8_t* oc;                          // requantized output (bits_out 4 / 8)
  float* os;
  unsigned long long phase;
  const unsigned long long* epoch;
};

__device__ __forceinline__ int take_ticket(unsigned long long* work) {
  __shared__ int s_t;
  if (threadIdx.x == 0) s_t = static_cast<int>(atomicAdd(work, 1ull));
  __syncthreads();
  return s_t;
}

// flags f[j * kMaxChunks] >= target for j < n (thread 0 spins, the CTA waits)
__device__ __forceinline__ void wait_flags(const unsigned long long* f, int n, unsigned long long target) {
  if (threadIdx.x == 0) {
    const unsigned long long t0 = globaltimer();
    for (int j = 0; j < n; ++j)
      while (ld_acquire_sys(f + static_cast<int64_t>(j) * kMaxChunks) < target)
        if (globaltimer() - t0 > 20000000000ull) __trap();
  }
  __syncthreads();
}

// producer CTA done with chunk c: the last of the gp producers publishes it
__device__ __forceinline__ void arrive(unsigned int* cnt, int c, int gp, unsigned long long* const* dst, int n,
                                       unsigned long long v, unsigned long long* dbg = nullptr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(cnt + c, 1u) == static_cast<unsigned>(gp) - 1u) {
      if (dbg) dbg[c * 4 + 3] = globaltimer();
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      for (int j = 0; j < n; ++j) st_relaxed_sys(dst[j] + c, v);
      if (dbg) dbg[c * 4 + 0] = globaltimer();
    }
  }
}

// the last CTA of the launch resets the ticket / exit / chunk counters
__device__ __forceinline__ void finish(unsigned long long* work, unsigned int* cnt, int nch) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(work + 1, 1ull) == gridDim.x - 1ull;
  }
  __syncthreads();
  if (s_last) {
    for (int c = threadIdx.x; c < nch; c += kThreads) cnt[c] = 0u;
    if (threadIdx.x == 0) {
      work[0] = 0ull;
      work[1] = 0ull;
    }
    __threadfence();
  }
}

// one warp item: quantize the U blocks starting at block blk0 (codes / scales at
// the same block offsets)
template <typename T, int BITS, int U = kU>
__device__ __forceinline__ void quantize_item(const T* __restrict__ x, int64_t blk0, uint8_t* __restrict__ codes,
                                              float* __restrict__ scales) {
  const int lane = threadIdx.x & 31;
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

// ------------------------------------------------------------------------ AG
template <typename T, int BITS, typename TO>
__global__ void __launch_bounds__(kThreads) k_ag_pipe(const __grid_constant__ FusedAG a,
                                                      const __grid_constant__ SyncArgs sy) {
  sync_wait(sy);   // every rank is done with the previous phase: our buffers are free
  const unsigned long long target = a.phase + (a.epoch ? *a.epoch : 0ull);
  const int ticket = take_ticket(a.work);
  const int w = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (a.dbg && ticket == 0 && threadIdx.x == 0) a.dbg[(kMaxChunks - 1) * 4] = globaltimer();
  if (ticket < a.gp) {                                    // producer
    const int64_t stride = static_cast<int64_t>(a.gp) * kWarps;
    const int64_t vw = static_cast<int64_t>(ticket) * kWarps + w;
    for (int c = 0; c < a.nch; ++c) {
      const int64_t e0 = c * a.C;
      const int64_t nit = min(a.C, a.plen - e0) / (kB * kU);
      for (int64_t it = vw; it < nit; it += stride)
        quantize_item<T, BITS>(static_cast<const T*>(a.x), e0 / kB + it * kU, a.qc, a.qs);
      arrive(a.cnt, c, a.gp, a.flags_remote, a.D, target, a.dbg);
    }
  } else {                                                // consumer
    const int64_t gc = static_cast<int64_t>(gridDim.x) - a.gp;
    const int64_t vw = static_cast<int64_t>(ticket - a.gp) * kWarps + w;
    const int64_t stride = gc * kWarps;
    TO* y = static_cast<TO*>(a.y);
    for (int c = 0; c < a.nch; ++c) {
      wait_flags(a.flags + c, a.D, target);               // chunk c published by every member
      if (a.dbg && threadIdx.x == 0) atomicMin(a.dbg + c * 4 + 1, globaltimer());
      const int64_t e0 = c * a.C;
      const int64_t nt = min(a.C, a.plen - e0) / (256 * kU);   // warp tiles per piece
      // tiles interleave the pieces: local (HBM) and peer (NVLink) tiles in flight together
      for (int64_t t = vw; t < nt * a.D; t += stride) {
        const int j = static_cast<int>((t + a.me + 1) % a.D);
        const int64_t eb = e0 + (t / a.D) * (256 * kU);
        Codes8<BITS> raw[kU];
        float sc[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int64_t e = eb + (u * 32 + lane) * 8;
          raw[u].load(a.pc[j] + e * BITS / 8);
          sc[u] = __ldg(a.ps[j] + e / kB);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int64_t e = eb + (u * 32 + lane) * 8;
          float cd[8], v[8];
          raw[u].decode(cd);
#pragma unroll
          for (int i = 0; i < 8; ++i) v[i] = __fmul_rn(cd[i], sc[u]);
          Out8<TO>::store(y + j * a.plen + e, v);
        }
      }
      if (a.dbg) {
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(a.dbg + c * 4 + 2, globaltimer());
      }
    }
  }
  finish(a.work, a.cnt, a.nch);
  sync_signal(sy);   // done(phase)
}

// ------------------------------------------------------------------------ RS
template <typename T, int BIN, int BOUT, int GT>
__global__ void __launch_bounds__(kThreads) k_rs_pipe(const __grid_constant__ FusedRS a,
                                                      const __grid_constant__ SyncArgs sy) {
  sync_wait(sy);
  const unsigned long long target = a.phase + (a.epoch ? *a.epoch : 0ull);
  const int ticket = take_ticket(a.work);
  const int w = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (ticket < a.gp) {                                    // producer: chunk c for every destination
    const int64_t stride = static_cast<int64_t>(a.gp) * kWarps;
    const int64_t vw = static_cast<int64_t>(ticket) * kWarps + w;
    for (int c = 0; c < a.ncl; ++c) {
      const int64_t off = c * a.C;
      const int64_t nit = min(a.C, a.cl - off) / (kB * kU);   // warp items per destination
      for (int64_t t = vw; t < nit * GT; t += stride) {
        const int dest = static_cast<int>(t % GT);
        quantize_item<T, BIN>(static_cast<const T*>(a.x), (dest * a.cl + off) / kB + (t / GT) * kU, a.qc, a.qs);
      }
      arrive(a.cnt, c, a.gp, a.flags_remote, GT, target);   // flag row d in member j's pool
    }
  } else {                                                // consumer: reduce chunk c destined here
    const int64_t gc = static_cast<int64_t>(gridDim.x) - a.gp;
    const int64_t vw = static_cast<int64_t>(ticket - a.gp) * kWarps + w;
    const int64_t stride = gc * kWarps;
    for (int c = 0; c < a.ncl; ++c) {
      wait_flags(a.flags + c, GT, target);
      const int64_t off = c * a.C;
      const int64_t nit = min(a.C, a.cl - off) / (kB * kU);
      for (int64_t it = vw; it < nit; it += stride) {
        const int64_t blk0 = off / kB + it * kU;
        Codes8<BIN> raw[kU][GT];
        float sc[kU][GT];
#pragma unroll
        for (int u = 0; u < kU; ++u)
#pragma unroll
          for (int p = 0; p < GT; ++p) {
            raw[u][p].load(a.mc[p] + ((blk0 + u) * kB + lane * 8) * BIN / 8);
            sc[u][p] = __ldg(a.ms[p] + blk0 + u);
          }
        float v[kU][1][8];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          float cd[8];
#pragma unroll
          for (int p = 0; p < GT; ++p) {
            raw[u][p].decode(cd);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float xh = __fmul_rn(cd[i], sc[u][p]);
              v[u][0][i] = p == 0 ? xh : __fadd_rn(v[u][0][i], xh);   // ascending member digit
            }
          }
        }
        if constexpr (BOUT == 0) {
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            float* dst = a.of + (blk0 + u) * kB + lane * 8;
            if (a.acc) {
              const float4 o0 = reinterpret_cast<const float4*>(dst)[0];
              const float4 o1 = reinterpret_cast<const float4*>(dst)[1];
              const float old[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
              for (int i = 0; i < 8; ++i) v[u][0][i] = __fadd_rn(old[i], v[u][0][i]);   // A = fl(A + P)
            }
            Out8<float>::store(dst, v[u][0]);
          }
        } else {
          float am[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            float m = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) m = fmaxf(m, fabsf(v[u][0][i]));
            am[u] = group_max<32>(m);
          }
          quantize_store<kB, BOUT, kU>(v, am, blk0, lane, a.oc, a.os);
        }
      }
    }
  }
  finish(a.work, a.cnt, a.ncl);
  sync_signal(sy);
}

// grid: SMs x resident CTAs; producers = pf % of it (HZ_TUNE pf, default 30)
int producers(int64_t grid) {
  int64_t gp = grid * tune_param("pf", 30) / 100;
  if (gp < 1) gp = 1;
  if (gp > grid - 1) gp = grid - 1;
  return static_cast<int>(gp);
}

int64_t pipe_grid(const void* kernel) {
  const int64_t g = grid_for(kernel, int64_t(1) << 40);   // capacity
  return g < 2 ? 2 : g;
}

template <typename T, int BITS, typename TO>
cudaError_t ag_t(FusedAG a, cudaStream_t st, const SyncArgs& sy) {
  auto kern = k_ag_pipe<T, BITS, TO>;
  const int64_t grid = pipe_grid(reinterpret_cast<const void*>(kern));
  a.gp = producers(grid);
  return launch_k(kern, grid, st, a, sy);
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
cudaError_t rs_t(FusedRS a, cudaStream_t st, const SyncArgs& sy) {
  auto kern = k_rs_pipe<T, BIN, BOUT, GT>;
  const int64_t grid = pipe_grid(reinterpret_cast<const void*>(kern));
  a.gp = producers(grid);
  return launch_k(kern, grid, st, a, sy);
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
  a.cnt = h.cnt;
  a.dbg = h.dbg;
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
  a.cnt = h.cnt;
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
