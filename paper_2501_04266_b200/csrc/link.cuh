// NVLink link CTAs: TMA bulk copies of peer buffers into a shared-memory ring, and
// the device-side work queue that balances the rest of a launch.  Internal header.
//
// Why: a peer read is a ~2 µs round trip over NVLink, so the link
// is filled only with ~1.5 MB in flight per GPU.  Plain vector loads need the whole
// grid for that (each warp holds a few KB), which ties every SM to the link for the
// whole launch.  A bulk copy (cp.async.bulk global -> shared, completion counted on an
// mbarrier) moves a 16 KB tile per instruction, so a few dozen "link CTAs" with a
// 3-stage ring each keep the link saturated (tools/bulk_probe.cu: 680-695 GB/s from
// 16-24 CTAs, against 484 GB/s for plain loads), and the remaining CTAs stream the
// HBM-bound work (local piece, quantize) from a shared atomic queue, which the link
// CTAs join when their peer tiles are done.
//
// Ordering: the launch's phase wait (sync_wait: thread 0 acquires the producers' flags
// at system scope, then bar.sync) precedes every bulk copy; the issuing thread then
// runs fence.proxy.async so that the async proxy's reads are ordered after that
// acquire.  A stage is re-armed only after every thread has consumed it (bar.sync),
// followed by a proxy fence for the generic-proxy reads -> async-proxy write order.
#pragma once

#include "codec.cuh"

namespace hz {
namespace dev {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
}
// bytes % 16 == 0, src / dst 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

// Shared-memory ring of S stages of `stage_bytes`, and its S mbarriers (one arrival:
// the issuing thread's expect_tx; the bulk copies complete the transaction count).
// Tile i of this CTA lives in stage i % S; its completion has parity (i / S) & 1.
struct Ring {
  char* buf;
  uint64_t* bar;
  int S;
  int stage_bytes;
  __device__ __forceinline__ char* stage(int64_t i) const { return buf + (i % S) * stage_bytes; }
  __device__ __forceinline__ uint64_t* full(int64_t i) const { return bar + (i % S); }
  __device__ __forceinline__ unsigned parity(int64_t i) const { return static_cast<unsigned>((i / S) & 1); }
};

// Run this CTA's `mine` tiles through the ring: issue(i, stage, bar) arms the barrier
// and starts the copies of tile i (thread 0 only); consume(i, stage) is run by every
// thread once the tile has landed.  Requires a ring initialised by ring_init.
template <class Issue, class Consume>
__device__ __forceinline__ void ring_run(const Ring& r, int64_t mine, Issue&& issue, Consume&& consume) {
  if (threadIdx.x == 0) {
    fence_proxy_async();
    for (int64_t i = 0; i < r.S && i < mine; ++i) issue(i, r.stage(i), r.full(i));
  }
  for (int64_t i = 0; i < mine; ++i) {
    mbar_wait(r.full(i), r.parity(i));
    consume(i, r.stage(i));
    __syncthreads();
    if (threadIdx.x == 0 && i + r.S < mine) {
      fence_proxy_async();
      issue(i + r.S, r.stage(i + r.S), r.full(i + r.S));
    }
  }
}

// The ring lives at the start of the dynamic shared memory: S stages, then S barriers.
__device__ __forceinline__ Ring ring_init(char* smem, int S, int stage_bytes) {
  Ring r{smem, reinterpret_cast<uint64_t*>(smem + S * stage_bytes), S, stage_bytes};
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(r.bar + s, 1);
    mbar_init_fence();
  }
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------- work queue
// queue[0]: next task; queue[1]: CTAs that have left the queue.  The last CTA to
// leave resets both (the launch after this one on the stream starts from 0; graph
// replays too).  Returns the CTA's next task index (the same value in every thread).
__device__ __forceinline__ int64_t queue_next(unsigned* queue, int* slot) {
  __syncthreads();   // every thread is done with the previous task's shared state
  if (threadIdx.x == 0) *slot = static_cast<int>(atomicAdd(queue, 1u));
  __syncthreads();
  return *slot;
}
__device__ __forceinline__ void queue_leave(unsigned* queue) {
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(queue + 1, 1u) == gridDim.x - 1) {
      queue[0] = 0u;
      queue[1] = 0u;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------ link gather tiles
// Gather+dequantize of the REMOTE pieces of pc (8-bit codes, B = 256, bf16 out) by
// the link CTAs: tile = up to te elements of one piece (te bytes of codes + te/64 of
// scales per stage); tiles of different pieces interleave (all peers' links busy).
// Ring geometry (host-chosen, HZ_TUNE lte / ls): te elements per tile (a multiple of
// 1024: te code bytes + te/64 scale bytes per stage), S stages (<= kLinkSMax).
constexpr int kLinkSMax = 4;
struct LinkGeo {
  int te;
  int S;
  __host__ __device__ __forceinline__ int stage() const { return te + te / 64; }
  __host__ __device__ __forceinline__ int smem() const { return S * stage() + S * 8; }
};

struct LinkTiles {
  int nrem;            // remote pieces
  int rj[kMaxWorld];   // their piece indices
  int64_t per;         // tiles per piece
  int te;              // elements per tile
  __device__ __forceinline__ int64_t count() const { return nrem * per; }
};

__device__ __forceinline__ LinkTiles link_tiles(const Pieces& pc, int te) {
  LinkTiles t{};
  for (int j = 0; j < pc.n; ++j)
    if ((pc.remote >> j) & 1u) t.rj[t.nrem++] = j;
  t.te = te;
  t.per = (pc.len + te - 1) / te;
  return t;
}

// remote tile t (0 <= t < count()): piece lt.rj[t % nrem], elements [e0, e0 + cnt)
__device__ __forceinline__ void link_tile(const Pieces& pc, const LinkTiles& lt, int64_t t, int& j, int64_t& e0,
                                          int64_t& cnt) {
  j = lt.rj[t % lt.nrem];
  e0 = (t / lt.nrem) * lt.te;
  cnt = pc.len - e0 < lt.te ? pc.len - e0 : lt.te;   // multiple of 1024 (Np % (W*4*B) == 0)
}

// thread 0: arm `bar` and start the bulk copies of remote tile t into `stage`
__device__ __forceinline__ void link_issue(const Pieces& pc, const LinkTiles& lt, int64_t t, char* stage,
                                           uint64_t* bar) {
  int j;
  int64_t e0, cnt;
  link_tile(pc, lt, t, j, e0, cnt);
  const unsigned cb = static_cast<unsigned>(cnt), sb = static_cast<unsigned>(cnt / 256 * 4);
  mbar_expect_tx(bar, cb + sb);
  bulk_g2s(stage, pc.c[j] + e0, cb, bar);
  bulk_g2s(stage + lt.te, pc.s[j] + e0 / 256, sb, bar);
}

// every thread: dequantize the landed remote tile t from `stage` into y (and the hpZ
// secondary range when pc.sec_c)
template <typename TO>
__device__ __forceinline__ void link_consume(const Pieces& pc, const LinkTiles& lt, int64_t t, const char* stage,
                                             TO* __restrict__ y) {
  int j;
  int64_t e0, cnt;
  link_tile(pc, lt, t, j, e0, cnt);
  const float* sc = reinterpret_cast<const float*>(stage + lt.te);
  const int64_t g0 = j * pc.len + e0;   // layer element of the tile's first code
  for (int u = threadIdx.x; u < cnt / 8; u += kThreads) {
    Codes8<8> raw;
    raw.r = *reinterpret_cast<const uint2*>(stage + u * 8);
    const float s = sc[u >> 5];
    float c[8], v[8];
    raw.decode(c);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __fmul_rn(c[k], s);
    const int64_t e = g0 + u * 8;
    Out8<TO>::store(y + e, v);
    if (pc.sec_c && e >= pc.sec_lo && e < pc.sec_hi) {
      raw.store(pc.sec_c + (e - pc.sec_lo));
      if (((e - pc.sec_lo) & 255) == 0) pc.sec_s[(e - pc.sec_lo) >> 8] = s;
    }
  }
}

// dedicated link CTA: remote tiles first, first + stride, ... through the ring
template <typename TO>
__device__ __forceinline__ void link_gather(const Pieces& pc, const LinkTiles& lt, TO* __restrict__ y,
                                            const Ring& ring, int64_t first, int64_t stride) {
  const int64_t total = lt.count();
  const int64_t mine = total > first ? (total - first + stride - 1) / stride : 0;
  ring_run(
      ring, mine,
      [&](int64_t i, char* stage, uint64_t* bar) { link_issue(pc, lt, first + i * stride, stage, bar); },
      [&](int64_t i, char* stage) { link_consume<TO>(pc, lt, first + i * stride, stage, y); });
}

}  // namespace dev
}  // namespace hz
