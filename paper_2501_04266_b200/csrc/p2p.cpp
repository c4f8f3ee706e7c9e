// NVLink peer-memory transport (hz_enable_p2p; hz_init_virtual): the per-level
// collectives are fused into the codec kernels instead of being staged through NCCL.
//
// Every rank owns one symmetric pool (cudaMalloc + cudaIpcGetMemHandle; the handles
// are exchanged with one ncclAllGather and opened with cudaIpcOpenMemHandle), so a
// buffer at pool offset X on this rank is at offset X in every peer's pool.
// Allocations (hz_sym_alloc and the library's slots) are bump allocations made in
// the same order on every rank, hence symmetric.
//
// qwZ/hpZ all-gather (O7/O8): the owner quantizes its primary into a pool buffer
// (the caller's pool-allocated secondary when s == w); each rank then runs ONE
// gather+dequantize kernel whose pieces are the members' codes, read straight over
// NVLink — the gathered codes never land in HBM.  Backward: the same kernel over
// the members' secondaries.
// qgZ reduce-scatter (O9): a hop's send buffer (the quantize output, or the previous
// hop's requantized sum) lives in the pool; the hop's reduce kernel reads the chunk
// destined to this rank from every member's send buffer over NVLink and sums in
// ascending member order — the all-to-all and the dequant+sum are one kernel.
//
// Ordering (codec.cuh): every call is one or more numbered phases, the same numbers
// on every rank.  Synchronisation is level-local (the devices involved in an
// exchange do not scale with the job):
//   * a kernel that READS peers' buffers produced in the same phase waits for
//     `ready >= phase` from exactly those peers (the gather members, the hop group);
//   * a kernel that OVERWRITES a pool buffer waits for `done >= phase-1` from the
//     ranks that read this rank's copy of that buffer in earlier calls (`readers`);
//   * a backward gather reads secondaries written in an earlier phase and waits for
//     `done >= phase-1` from its members (every rank finished every earlier phase);
//   * the kernel that completes a phase signals `done(phase)` to `nbr`, the ranks this
//     rank reads from (and, from a forward gather on, the members of its backward
//     gather): `done[q] >= v` at a rank certifies that q finished all its reads and
//     writes of phases <= v.  Producers signal `ready(phase)` to the readers of what
//     they wrote.
// So a pair exchange waits only for the pair, whatever the other ranks do.  All P2P
// calls of one context must be issued on one stream, in the same order on every rank
// (the NCCL discipline).
//
// Paired layers (hz_allgather_params_next / hz_backward_step): one dual kernel
// (k_gather_quantize) runs a gather of phase a and a quantize of phase a+1.  It waits
// for its gather's condition and for `done >= a-1` from the readers of what the
// quantize overwrites, and signals done(a) and ready(a+1).  A prefetched quantize
// whose layer is not gathered next (another call comes first) leaves phase a+1
// without a `done`; flush_prefetch completes it before the next phase starts.
//
// Virtual world (hz_init_virtual, vworld.cpp): W contexts in one process on one GPU,
// whose peer pools are each other's allocations.  The same kernels and flags run;
// in addition every launch is ordered on the host after the launches that signal
// what it waits for (CUDA events), so the W streams cannot deadlock on shared
// hardware queues or SMs.
#include <algorithm>
#include <mutex>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "ctx.h"

namespace hz {
namespace {

#define P2P_CUDA(call, what)                              \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(e_, what);    \
  } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

hz_status pool_alloc(hz_ctx* ctx, size_t bytes, size_t* off) {
  auto& P = ctx->p2p;
  const size_t o = align_up(P.used, 256);
  if (o + bytes > P.bytes)
    return fail(HZ_ERR_INVALID, "P2P pool exhausted: need " + std::to_string(o + bytes) + " of " +
                                    std::to_string(P.bytes) + " bytes (pass a larger pool_bytes)");
  *off = o;
  P.used = o + bytes;
  return HZ_OK;
}

hz_status slot(hz_ctx* ctx, hz_ctx::P2P::Slot& sl, size_t bytes) {
  if (sl.cap >= bytes) return HZ_OK;
  hz_status rc = pool_alloc(ctx, bytes, &sl.off);
  if (rc == HZ_OK) sl.cap = bytes;
  return rc;
}

template <typename T>
T* at(hz_ctx* ctx, int q, size_t off) {
  return reinterpret_cast<T*>(ctx->p2p.peer[q] + off);
}

size_t off_of(const hz_ctx* ctx, const void* local) {
  return static_cast<size_t>(static_cast<const char*>(local) - ctx->p2p.pool);
}

unsigned mask_of(const std::vector<int>& ranks, int me) {
  unsigned m = 0;
  for (int r : ranks)
    if (r != me) m |= 1u << r;
  return m;
}

// readers of this rank's copy of the pool buffer at `local` (earlier calls)
unsigned readers_of(const hz_ctx* ctx, const void* local) {
  auto it = ctx->p2p.readers.find(off_of(ctx, local));
  return it == ctx->p2p.readers.end() ? 0u : it->second;
}

void add_readers(hz_ctx* ctx, const void* local, unsigned m) { ctx->p2p.readers[off_of(ctx, local)] |= m; }

// Phase arguments are absolute phase numbers; the kernel sees them relative to the
// device epoch (graph replays advance it).  A zero mask disables that wait / signal.
struct Phases {
  unsigned long long wr = 0, wd = 0, sr = 0, sd = 0;
  unsigned wr_mask = 0, wd_mask = 0, sr_mask = 0, sd_mask = 0;
};

SyncArgs make_sync(hz_ctx* ctx, const Phases& ph) {
  auto& P = ctx->p2p;
  SyncArgs s{};
  s.ready_local = reinterpret_cast<unsigned long long*>(P.pool + kReadyOff);
  s.done_local = reinterpret_cast<unsigned long long*>(P.pool + kDoneOff);
  for (int q = 0; q < ctx->world; ++q) {
    s.ready_remote[q] = reinterpret_cast<unsigned long long*>(P.peer[q] + kReadyOff) + ctx->rank;
    s.done_remote[q] = reinterpret_cast<unsigned long long*>(P.peer[q] + kDoneOff) + ctx->rank;
  }
  s.counter = reinterpret_cast<unsigned int*>(P.pool + kCounterOff);
  s.epoch = reinterpret_cast<const unsigned long long*>(P.pool + kEpochOff);
  s.abort = P.abort_dev;
  s.timeout_ns = P.timeout_ns;
  const unsigned long long e = P.epoch_host;
  s.wait_ready = ph.wr - e;
  s.wait_done = ph.wd - e;
  s.sig_ready = ph.sr - e;
  s.sig_done = ph.sd - e;
  s.wr_mask = ph.wr_mask;
  s.wd_mask = ph.wd_mask;
  s.sr_mask = ph.sr_mask;
  s.sd_mask = ph.sd_mask;
  return s;
}

// One synchronised launch: in a virtual world the host first orders the stream after
// the signals this kernel waits for, and records its own signals afterwards.
// (HZ_TUNE vworder=0 disables the host ordering: a test of the device-side waits)
// HZ_TUNE vwserial=1 (profiling tool mode, tools/vw_profile.py under ncu): in a virtual
// world, one synchronised launch at a time in the whole process, each completed before
// the next starts — so a profiler replaying one GPU's kernel (and restoring that GPU's
// memory between passes) never races a peer kernel writing flags into that memory.
std::mutex g_vw_serial;

template <class F>
hz_status synced(hz_ctx* ctx, const SyncArgs& s, cudaStream_t st, F&& launch) {
  static const bool order = tune_param("vworder", 1) != 0;
  static const bool serial = tune_param("vwserial", 0) != 0;
  const bool vw = ctx->p2p.vw && order;
  hz_status rc;
  if (vw && (rc = vw_wait(ctx, s, st)) != HZ_OK) return rc;
  if (vw && serial) {
    std::lock_guard<std::mutex> lock(g_vw_serial);
    if ((rc = launch()) != HZ_OK) return rc;
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "virtual world: serial launch");
    return vw_signal(ctx, s, st);
  }
  if ((rc = launch()) != HZ_OK) return rc;
  if (vw) return vw_signal(ctx, s, st);
  return HZ_OK;
}

// Members of this rank's cumulative group of `level` (ranks that share every digit
// above `level`), as (off_level within range_0, rank), sorted by offset: piece k of
// the gathered layer is owned by the k-th entry.
std::vector<std::pair<int64_t, int>> cumulative_members(const hz_partition_t* p, int level) {
  std::vector<int> ranks;
  std::vector<int64_t> rel;
  std::vector<std::pair<int64_t, int>> out;
  if (level < 1) {
    out.emplace_back(0, p->rank);
    return out;
  }
  hop_members(p, 1, level, &ranks, &rel, nullptr);
  for (size_t k = 0; k < ranks.size(); ++k) out.emplace_back(rel[k], ranks[k]);
  std::sort(out.begin(), out.end());
  return out;
}

unsigned mask_of(const std::vector<std::pair<int64_t, int>>& mem, int me) {
  unsigned m = 0;
  for (const auto& x : mem)
    if (x.second != me) m |= 1u << x.second;
  return m;
}

}  // namespace

hz_status p2p_check(const hz_ctx* ctx) {
  const auto& P = ctx->p2p;
  if (P.abort_host && *reinterpret_cast<volatile unsigned*>(P.abort_host))
    return fail(HZ_ERR_ABORTED, "context aborted: a cross-GPU wait timed out or hz_abort was called "
                                "(only hz_finalize is allowed now)");
  return HZ_OK;
}

// A prefetched quantize (hz_allgather_params_next) whose layer is not gathered next
// leaves its phase without a `done`; complete it before any other phase starts: a
// one-CTA kernel signalling done(pre_phase) — nobody reads those codes in that phase,
// and every earlier read of this rank is complete in stream order.
// The deferred last qgZ hop of the previous hz_backward_step, as its own launch (when
// the next call cannot carry it): waits for the hop's inputs (ready >= its phase from
// the hop group) and signals done(its phase) — no phase was issued since.
hz_status flush_reduce(hz_ctx* ctx, cudaStream_t st) {
  auto& P = ctx->p2p;
  if (!P.pend.on) return HZ_OK;
  const auto r = P.pend;
  P.pend.on = false;
  Phases f;
  f.wr = r.ph;
  f.wr_mask = r.wr_mask;
  f.sd = r.ph;
  f.sd_mask = P.nbr;
  SyncArgs sr = make_sync(ctx, f);
  return synced(ctx, sr, st, [&] {
    return run_reduce(r.g, r.c, r.s, r.n, r.bits, r.block, 0, nullptr, nullptr, r.shard, r.acc, st, r.level, &sr,
                      r.remote);
  });
}

hz_status flush_prefetch(hz_ctx* ctx, cudaStream_t st, bool keep_reduce = false) {
  auto& P = ctx->p2p;
  // (a deferred reduce and a prefetched quantize are never pending together: each
  // call flushes the other kind on entry; flags stay monotone)
  if (!keep_reduce) {
    hz_status rc = flush_reduce(ctx, st);
    if (rc != HZ_OK) return rc;
  }
  if (!P.pre_phase) return HZ_OK;
  const unsigned long long ph = P.pre_phase;
  P.pre_phase = 0;
  P.pre_codes = P.pre_primary = nullptr;
  Pieces pc{};
  pc.n = 1;
  Phases f;
  f.sd = ph;
  f.sd_mask = P.nbr;
  SyncArgs s = make_sync(ctx, f);
  return synced(ctx, s, st, [&] { return run_gather_dequantize(pc, 0, 8, 256, nullptr, HZ_BF16, st, 0, &s, 0); });
}

bool in_pool(const hz_ctx* ctx, const void* p, size_t bytes) {
  const char* c = static_cast<const char*>(p);
  return ctx->p2p.on && c >= ctx->p2p.pool + kPoolHeader && c + bytes <= ctx->p2p.pool + ctx->p2p.bytes;
}

bool p2p_next_fusable(const hz_ctx* ctx, const hz_partition_t* p, int bits, hz_dtype out_dt, const NextQ& nx) {
  const hz_partition_t* q = nx.p;
  return ctx->p2p.on && q && p->s == p->w && q->s == q->w && p->block == 256 && q->block == 256 &&
         gather_quantize_supported(256, bits, out_dt) && q->len[q->w] > 0 &&
         in_pool(ctx, nx.codes, code_bytes(q->len[q->s], bits)) && in_pool(ctx, nx.scales, q->len[q->s] / 256 * 4) &&
         tune_param("nofuse", 0) == 0;
}

hz_status p2p_allgather(hz_ctx* ctx, const hz_partition_t* p, int backward, const void* primary,
                        hz_dtype dt, int bits, uint8_t* sec_codes, float* sec_scales, void* full_out,
                        hz_dtype out_dt, cudaStream_t st, const NextQ* next) {
  auto& P = ctx->p2p;
  const int64_t Np = p->padded_numel;
  const int B = p->block;
  const int w = p->w, s = p->s;
  const int top = backward ? s : w;
  const int64_t len_s = p->len[s];
  if (!in_pool(ctx, sec_codes, code_bytes(len_s, bits)) || !in_pool(ctx, sec_scales, len_s / B * 4))
    return fail(HZ_ERR_INVALID, "sec_codes/sec_scales: must be hz_sym_alloc memory when P2P is enabled");
  hz_status rc;
  const auto members = cumulative_members(p, top);
  const int D = static_cast<int>(members.size());
  if (D > kMaxWorld) return fail(HZ_ERR_UNSUPPORTED, "P2P gather over more than 8 ranks");
  const unsigned gmask = mask_of(members, ctx->rank);                         // read in this call
  const unsigned smask = mask_of(cumulative_members(p, s), ctx->rank);        // backward group
  // this layer's primary already quantized by the previous call's dual kernel (the
  // prefetch of hz_allgather_params_next), in phase pre_phase, with no phase since,
  // from the same primary with the same code width, dtype and length
  const bool pre = !backward && s == w && P.pre_phase != 0 && P.pre_phase == P.phase && P.pre_codes == sec_codes &&
                   P.pre_primary == primary && P.pre_bits == bits && P.pre_dt == dt && P.pre_len == p->len[w];
  if (pre) {
    P.pre_phase = 0;
    P.pre_codes = P.pre_primary = nullptr;
    if ((rc = flush_reduce(ctx, st)) != HZ_OK) return rc;
  } else if ((rc = flush_prefetch(ctx, st)) != HZ_OK) {
    return rc;
  }
  // every call is a phase, even without peers to read from: it may write a secondary
  // that peers read in a later backward phase, and its done(phase) tells them so
  const unsigned long long phase = pre ? P.phase : ++P.phase;
  // the members read this rank's buffers from now on, and will gather its secondary
  // in the backward: they get this rank's `done` signals
  P.nbr |= gmask | smask;
  const int64_t plen = p->len[top];

  const uint8_t* xc;
  const float* xs;
  if (!backward) {
    uint8_t* qc = sec_codes;
    float* qs = sec_scales;
    if (s != w) {   // the quantized primary needs its own peer-readable buffer
      if ((rc = slot(ctx, P.ag_prim_c, code_bytes(p->len[w], 8))) != HZ_OK) return rc;
      if ((rc = slot(ctx, P.ag_prim_s, p->len[w] / B * 4)) != HZ_OK) return rc;
      qc = at<uint8_t>(ctx, ctx->rank, P.ag_prim_c.off);
      qs = at<float>(ctx, ctx->rank, P.ag_prim_s.off);
    }
    if (!pre) {
      // A2: overwrites qc (read by the gather members of earlier calls) and, in this
      // call, the secondary (read by the backward group)
      Phases f;
      f.wd = phase - 1;
      f.wd_mask = readers_of(ctx, qc) | readers_of(ctx, sec_codes);
      f.sr = phase;
      f.sr_mask = gmask;
      SyncArgs sq = make_sync(ctx, f);
      if ((rc = synced(ctx, sq, st, [&] { return run_quantize(primary, dt, p->len[w], bits, B, qc, qs, st, w, &sq); })) !=
          HZ_OK)
        return rc;
    }
    add_readers(ctx, qc, gmask);
    add_readers(ctx, sec_codes, smask);
    if (s > w) {   // A4, s > w: the secondary is a sub-slice of the own quantized primary
      const int64_t rel = p->off[s] - p->off[w];
      if ((rc = copy_async(sec_codes, qc + code_bytes(rel, bits), code_bytes(len_s, bits), st)) != HZ_OK) return rc;
      if ((rc = copy_async(sec_scales, qs + rel / B, len_s / B * 4, st)) != HZ_OK) return rc;
    }
    xc = qc;
    xs = qs;
  } else {
    xc = sec_codes;
    xs = sec_scales;
  }
  Pieces pc{};
  pc.n = D;
  pc.len = plen;
  int64_t remote = 0;
  for (int k = 0; k < D; ++k) {
    const int m = members[k].second;
    pc.c[k] = at<const uint8_t>(ctx, m, off_of(ctx, xc));
    pc.s[k] = at<const float>(ctx, m, off_of(ctx, xs));
    if (m != ctx->rank) remote += code_bytes(plen, bits) + plen / B * 4;
  }
  if (!backward && s < w) {   // A4, s < w: keep range_s of the gathered codes
    pc.sec_c = sec_codes;
    pc.sec_s = sec_scales;
    pc.sec_lo = p->off[s];
    pc.sec_hi = p->off[s] + len_s;
  }
  if (!backward && next && next->codes != sec_codes && next->scales != sec_scales &&
      p2p_next_fusable(ctx, p, bits, out_dt, *next)) {
    // gather this layer (phase) || quantize the next layer's primary (phase + 1) in one
    // launch.  Waits: the members' codes of this phase are ready, and the readers of
    // the next layer's secondary (earlier calls) are done.  Signals done(phase) and
    // ready(phase + 1) to the next layer's gather members.
    const unsigned long long nph = ++P.phase;
    const hz_partition_t* q = next->p;
    const unsigned nmask = mask_of(cumulative_members(q, q->w), ctx->rank);
    Phases f;
    f.wr = phase;
    f.wr_mask = gmask;
    f.wd = phase - 1;
    f.wd_mask = readers_of(ctx, next->codes);
    f.sd = phase;
    f.sd_mask = P.nbr;
    f.sr = nph;
    f.sr_mask = nmask;
    SyncArgs sd = make_sync(ctx, f);
    if ((rc = synced(ctx, sd, st, [&] {
           return run_gather_quantize(pc, Np, bits, full_out, out_dt, next->primary, dt, q->len[q->w], bits,
                                      next->codes, next->scales, st, sd, remote);
         })) != HZ_OK)
      return rc;
    P.pre_phase = nph;
    P.pre_codes = next->codes;
    P.pre_primary = next->primary;
    P.pre_bits = bits;
    P.pre_dt = dt;
    P.pre_len = q->len[q->w];
    clear_error();
    return HZ_OK;
  }
  Phases f;
  if (backward) {   // secondaries written in earlier phases: the members finished them
    f.wd = phase - 1;
    f.wd_mask = gmask;
  } else {
    f.wr = phase;
    f.wr_mask = gmask;
  }
  f.sd = phase;
  f.sd_mask = P.nbr;
  SyncArgs sd = make_sync(ctx, f);
  if ((rc = synced(ctx, sd, st, [&] { return run_gather_dequantize(pc, Np, bits, B, full_out, out_dt, st, 0, &sd, remote); })) !=
      HZ_OK)
    return rc;
  clear_error();
  return HZ_OK;
}

bool p2p_prev_fusable(const hz_ctx* ctx, const hz_partition_t* p, int from_level, const PrevG& pg) {
  const hz_partition_t* q = pg.p;
  return ctx->p2p.on && q && p->block == 256 && q->block == 256 && p->len[from_level - 1] > 0 &&
         gather_quantize_supported(256, pg.bits, pg.out_dt) &&
         in_pool(ctx, pg.sec_codes, code_bytes(q->len[q->s], pg.bits)) &&
         in_pool(ctx, pg.sec_scales, q->len[q->s] / 256 * 4) &&
         static_cast<int>(cumulative_members(q, q->s).size()) <= kMaxWorld && tune_param("nofuse", 0) == 0;
}

hz_status p2p_reduce_scatter(hz_ctx* ctx, const hz_partition_t* p, const void* grad, hz_dtype dt,
                             int from_level, int to_level, const int* bits_per_level, float* shard,
                             int accumulate, cudaStream_t st, const PrevG* prev) {
  auto& P = ctx->p2p;
  const int B = p->block;
  hz_status rc;
  std::vector<Hop> hops;
  if ((rc = hops_of(p, from_level, to_level, &hops)) != HZ_OK) return rc;
  const int H = static_cast<int>(hops.size());
  // members of every hop (ascending rank), the offset of each member's chunk in the
  // hop's input range, and this rank's index
  std::vector<std::vector<int>> hr(H);
  std::vector<std::vector<int64_t>> hrel(H);
  std::vector<int> hme(H, 0);
  std::vector<unsigned> hmask(H, 0u);
  for (int h = 0; h < H; ++h) {
    hop_members(p, hops[h].a, hops[h].b, &hr[h], &hrel[h], &hme[h]);
    if (static_cast<int>(hr[h].size()) > kMaxG) return fail(HZ_ERR_UNSUPPORTED, "more than 16 ranks in one qgZ hop");
    hmask[h] = mask_of(hr[h], ctx->rank);
  }
  // a deferred hop of the previous call rides in this call's first launch when that is a
  // backward triple kernel (prev given, the pending reduce of the supported shape);
  // otherwise it is flushed as its own launch first
  const bool carry = prev && P.pend.on &&
                     gather_quantize_reduce_supported(prev->bits, prev->out_dt, P.pend.g, P.pend.bits) &&
                     P.pend.block == 256 && tune_param("defer", 1) != 0;
  if ((rc = flush_prefetch(ctx, st, carry)) != HZ_OK) return rc;
  // hop send buffers (8-bit capacity), indexed by the first level.  The last hop's input
  // alternates between two buffers per call (a deferred last hop of the previous call
  // still reads the other one); the other hops' buffers are single
  const int par = P.rs_par;
  P.rs_par ^= 1;
  auto bi = [&](int h) { return h == H - 1 ? par : 0; };
  for (int h = 0; h < H; ++h) {
    const Hop& hp = hops[h];
    if ((rc = slot(ctx, P.rs_c[hp.a][bi(h)], code_bytes(p->len[hp.a - 1], 8))) != HZ_OK) return rc;
    if ((rc = slot(ctx, P.rs_s[hp.a][bi(h)], p->len[hp.a - 1] / B * 4)) != HZ_OK) return rc;
  }
  // the previous layer's backward gather (phase gph) fused into this call's first
  // quantize (hz_backward_step; the caller checked p2p_prev_fusable)
  unsigned long long gph = 0;
  Pieces gpc{};
  int64_t gremote = 0;
  unsigned pmask = 0;
  if (prev) {
    gph = ++P.phase;
    const hz_partition_t* q = prev->p;
    const auto members = cumulative_members(q, q->s);
    pmask = mask_of(members, ctx->rank);
    gpc.n = static_cast<int>(members.size());
    gpc.len = q->len[q->s];
    for (int k = 0; k < gpc.n; ++k) {
      const int m = members[k].second;
      gpc.c[k] = at<const uint8_t>(ctx, m, off_of(ctx, prev->sec_codes));
      gpc.s[k] = at<const float>(ctx, m, off_of(ctx, prev->sec_scales));
      if (m != ctx->rank) gremote += code_bytes(gpc.len, prev->bits) + gpc.len / 256 * 4;
    }
  }
  const unsigned long long base = P.phase;
  P.phase += static_cast<unsigned long long>(H);
  auto phase_of = [&](int h) { return base + static_cast<unsigned long long>(h + 1); };
  for (int h = 0; h < H; ++h) P.nbr |= hmask[h];
  P.nbr |= pmask;

  uint8_t* c0 = at<uint8_t>(ctx, ctx->rank, P.rs_c[hops[0].a][bi(0)].off);
  float* s0 = at<float>(ctx, ctx->rank, P.rs_s[hops[0].a][bi(0)].off);
  const unsigned rb0 = readers_of(ctx, c0);
  add_readers(ctx, c0, hmask[0]);
  if (prev) {
    // previous layer's backward gather (phase gph) || A7 of this layer (phase gph + 1):
    // the previous layer's members finished every earlier phase (their secondaries are
    // complete) and the readers of the send buffer are done; signals done(gph) and
    // ready(gph + 1) to the first hop
    Phases f;
    f.wd = gph - 1;
    f.wd_mask = pmask | rb0;
    f.sd = gph;
    f.sd_mask = P.nbr;
    f.sr = phase_of(0);
    f.sr_mask = hmask[0];
    if (carry) {
      // + the previous call's deferred last hop (phase pend.ph = gph - 1): also wait for
      // its inputs (ready >= pend.ph from its hop group); done(gph) covers its phase.  The
      // done-wait drops to pend.ph - 1: the members' deferred phase completes only in
      // their own triple kernel (this same launch, on their side), and everything the
      // wait protects — the previous layer's secondaries, the last reads of the send
      // buffer c0 (the previous call's hops, or the launch before for the alternating
      // buffer) — completed in phases <= pend.ph - 1
      const auto r = P.pend;
      P.pend.on = false;
      f.wd = r.ph - 1;
      f.wr = r.ph;
      f.wr_mask = r.wr_mask;
      SyncArgs sq = make_sync(ctx, f);
      if ((rc = synced(ctx, sq, st, [&] {
             return run_gather_quantize_reduce(gpc, prev->p->padded_numel, prev->full_out, grad, dt,
                                               p->len[from_level - 1], bits_per_level[from_level - 1], c0, s0,
                                               r.g, r.c, r.s, r.n, r.bits, r.shard, r.acc, r.level, st, sq,
                                               gremote + r.remote);
           })) != HZ_OK)
        return rc;
    } else {
      SyncArgs sq = make_sync(ctx, f);
      if ((rc = synced(ctx, sq, st, [&] {
             return run_gather_quantize(gpc, prev->p->padded_numel, prev->bits, prev->full_out, prev->out_dt, grad,
                                        dt, p->len[from_level - 1], bits_per_level[from_level - 1], c0, s0, st, sq,
                                        gremote);
           })) != HZ_OK)
        return rc;
    }
  } else {
    // A7: quantize the input range_{from-1} into this rank's first send buffer
    Phases f;
    f.wd = phase_of(0) - 1;
    f.wd_mask = rb0;
    f.sr = phase_of(0);
    f.sr_mask = hmask[0];
    SyncArgs sq = make_sync(ctx, f);
    if ((rc = synced(ctx, sq, st, [&] {
           return run_quantize(grad, dt, p->len[from_level - 1], bits_per_level[from_level - 1], B, c0, s0, st,
                               from_level, &sq);
         })) != HZ_OK)
      return rc;
  }
  for (int h = 0; h < H; ++h) {
    const Hop& hp = hops[h];
    const int g = static_cast<int>(hr[h].size());
    const int bits = bits_per_level[hp.a - 1];
    const int64_t cl = p->len[hp.b];
    const int64_t my_rel = hrel[h][hme[h]];   // where this rank's chunk lies in every member's buffer
    const uint8_t* ptr_c[kMaxG];
    const float* ptr_s[kMaxG];
    for (int j = 0; j < g; ++j) {   // A8+A9: this rank's chunk of member j's send buffer, over NVLink
      ptr_c[j] = at<const uint8_t>(ctx, hr[h][j], P.rs_c[hp.a][bi(h)].off) + code_bytes(my_rel, bits);
      ptr_s[j] = at<const float>(ctx, hr[h][j], P.rs_s[hp.a][bi(h)].off) + my_rel / B;
    }
    const unsigned long long ph = phase_of(h);
    const int64_t remote = (g - 1) * (code_bytes(cl, bits) + cl / B * 4);
    Phases f;
    f.wr = ph;
    f.wr_mask = hmask[h];
    f.sd = ph;
    f.sd_mask = P.nbr;
    if (h + 1 < H) {
      uint8_t* oc = at<uint8_t>(ctx, ctx->rank, P.rs_c[hops[h + 1].a][bi(h + 1)].off);
      float* os = at<float>(ctx, ctx->rank, P.rs_s[hops[h + 1].a][bi(h + 1)].off);
      f.wd = ph - 1;
      f.wd_mask = readers_of(ctx, oc);
      add_readers(ctx, oc, hmask[h + 1]);
      f.sr = ph + 1;
      f.sr_mask = hmask[h + 1];
      SyncArgs sr = make_sync(ctx, f);
      if ((rc = synced(ctx, sr, st, [&] {
             return run_reduce(g, ptr_c, ptr_s, cl, bits, B, bits_per_level[hops[h + 1].a - 1], oc, os, nullptr, 0, st,
                               hp.b, &sr, remote);
           })) != HZ_OK)
        return rc;
    } else if (prev && B == 256 && tune_param("defer", 1) != 0) {
      // hz_backward_step: defer the last hop (fp32 shard) into the next call's launch —
      // the next layer's backward triple kernel (or a standalone flush)
      auto& r = P.pend;
      r.on = true;
      r.g = g;
      for (int j = 0; j < g; ++j) {
        r.c[j] = ptr_c[j];
        r.s[j] = ptr_s[j];
      }
      r.n = cl;
      r.bits = bits;
      r.block = B;
      r.shard = shard;
      r.acc = accumulate;
      r.level = hp.b;
      r.ph = ph;
      r.wr_mask = hmask[h];
      r.remote = remote;
    } else {
      SyncArgs sr = make_sync(ctx, f);
      if ((rc = synced(ctx, sr, st, [&] {
             return run_reduce(g, ptr_c, ptr_s, cl, bits, B, 0, nullptr, nullptr, shard, accumulate, st, hp.b, &sr,
                               remote);
           })) != HZ_OK)
        return rc;
    }
  }
  clear_error();
  return HZ_OK;
}

// A10 paper-literal option over NVLink: copy the shard into a peer-readable
// slot, then per level every rank reads all members' buffers in place and sums them
// in ascending digit (a full allreduce: each rank moves (g-1) * len bytes per level,
// twice the reduce-scatter's), and finally keeps its range_to slice.
hz_status p2p_allreduce_select(hz_ctx* ctx, const hz_partition_t* p, const float* in, int from_level, int to_level,
                               float* out, cudaStream_t st) {
  auto& P = ctx->p2p;
  hz_status rc;
  if ((rc = flush_prefetch(ctx, st)) != HZ_OK) return rc;
  const int64_t n = p->len[from_level - 1];
  const int64_t sel = p->off[to_level] - p->off[from_level - 1];
  if ((rc = slot(ctx, P.ar_a, n * 4)) != HZ_OK) return rc;
  if ((rc = slot(ctx, P.ar_b, n * 4)) != HZ_OK) return rc;
  std::vector<unsigned> lmask(HZ_MAX_LEVELS + 2, 0u);
  std::vector<std::vector<int>> lr(HZ_MAX_LEVELS + 2);
  for (int l = from_level; l <= to_level; ++l) {
    std::vector<int64_t> rel;
    hop_members(p, l, l, &lr[l], &rel, nullptr);
    lmask[l] = mask_of(lr[l], ctx->rank);
    P.nbr |= lmask[l];
  }
  const size_t off[2] = {P.ar_a.off, P.ar_b.off};
  const unsigned long long base = P.phase;
  P.phase += static_cast<unsigned long long>(to_level - from_level + 1);
  {   // copy-in (producer of phase base+1)
    Pieces pc{};
    pc.n = 1;
    pc.len = n;
    pc.c[0] = reinterpret_cast<const uint8_t*>(in);
    float* dst = at<float>(ctx, ctx->rank, off[0]);
    Phases f;
    f.wd = base;
    f.wd_mask = readers_of(ctx, dst);
    f.sr = base + 1;
    f.sr_mask = lmask[from_level];
    SyncArgs sq = make_sync(ctx, f);
    if ((rc = synced(ctx, sq, st, [&] { return run_sum(pc, n, dst, st, from_level, &sq, 0); })) != HZ_OK) return rc;
  }
  int cur = 0;
  for (int l = from_level; l <= to_level; ++l) {
    const int g = static_cast<int>(lr[l].size());
    const unsigned long long ph = base + static_cast<unsigned long long>(l - from_level + 1);
    Pieces pc{};
    pc.n = g;
    pc.len = n;
    int64_t remote = 0;
    for (int j = 0; j < g; ++j) {
      pc.c[j] = at<const uint8_t>(ctx, lr[l][j], off[cur]);
      if (lr[l][j] != ctx->rank) remote += n * 4;
    }
    float* dst = at<float>(ctx, ctx->rank, off[cur ^ 1]);
    Phases f;
    f.wr = ph;
    f.wr_mask = lmask[l];
    f.wd = ph - 1;
    f.wd_mask = readers_of(ctx, dst);
    add_readers(ctx, at<float>(ctx, ctx->rank, off[cur]), lmask[l]);
    f.sd = ph;
    f.sd_mask = P.nbr;
    if (l < to_level) {
      f.sr = ph + 1;
      f.sr_mask = lmask[l + 1];
    }
    SyncArgs sr = make_sync(ctx, f);
    if ((rc = synced(ctx, sr, st, [&] { return run_sum(pc, n, dst, st, l, &sr, remote); })) != HZ_OK) return rc;
    cur ^= 1;
  }
  // select range_to (local; the slot's next writer waits for this rank's readers)
  if ((rc = copy_async(out, at<float>(ctx, ctx->rank, off[cur]) + sel, static_cast<size_t>(p->len[to_level]) * 4,
                       st)) != HZ_OK)
    return rc;
  clear_error();
  return HZ_OK;
}

// Step tail over NVLink: AdamW writes the updated weights of range_L into a pool
// slot (producer), then one copy kernel gathers the members' slots — the ranks that
// share digits 1..w — into the primary range_w (consumer).
hz_status p2p_adamw_gather(hz_ctx* ctx, const hz_partition_t* p, const float* g, float* th, float* m, float* v,
                           const AdamW& hp, void* primary, hz_dtype dt, cudaStream_t st) {
  auto& P = ctx->p2p;
  const int L = p->levels, w = p->w;
  const int64_t lenL = p->len[L];
  const int64_t eb = elem_bytes(dt);
  hz_status rc;
  if ((rc = flush_prefetch(ctx, st)) != HZ_OK) return rc;
  if ((rc = slot(ctx, P.upd, lenL * 4)) != HZ_OK) return rc;   // fp32 capacity
  // members: vary digits w+1..L, keep digits 1..w; piece order = offset in range_w
  std::vector<int> hr;
  std::vector<int64_t> rel;
  std::vector<std::pair<int64_t, int>> mem;
  if (w < L) {
    hop_members(p, w + 1, L, &hr, &rel, nullptr);
    for (size_t k = 0; k < hr.size(); ++k) mem.emplace_back(rel[k], hr[k]);
    std::sort(mem.begin(), mem.end());
  } else {
    mem.emplace_back(0, ctx->rank);
  }
  std::vector<int> ranks;
  for (const auto& x : mem) ranks.push_back(x.second);
  const int D = static_cast<int>(ranks.size());
  if (D > kMaxWorld) return fail(HZ_ERR_UNSUPPORTED, "P2P gather over more than 8 ranks");
  const unsigned mmask = mask_of(ranks, ctx->rank);
  const unsigned long long phase = ++P.phase;
  P.nbr |= mmask;
  char* mine = at<char>(ctx, ctx->rank, P.upd.off);
  {
    Phases f;
    f.wd = phase - 1;
    f.wd_mask = readers_of(ctx, mine);
    f.sr = phase;
    f.sr_mask = mmask;
    SyncArgs sq = make_sync(ctx, f);
    if ((rc = synced(ctx, sq, st, [&] { return run_adamw(g, th, m, v, mine, dt, lenL, hp, st, &sq); })) != HZ_OK)
      return rc;
  }
  add_readers(ctx, mine, mmask);
  Pieces pc{};
  pc.n = D;
  pc.len = lenL * eb;   // bytes
  int64_t remote = 0;
  for (int k = 0; k < D; ++k) {
    pc.c[k] = at<const uint8_t>(ctx, ranks[k], P.upd.off);
    if (ranks[k] != ctx->rank) remote += pc.len;
  }
  Phases f;
  f.wr = phase;
  f.wr_mask = mmask;
  f.sd = phase;
  f.sd_mask = P.nbr;
  SyncArgs sd = make_sync(ctx, f);
  return synced(ctx, sd, st, [&]() -> hz_status {
    TraceScope t(st, "gather_copy", w, 16, lenL * D, D * pc.len * 2 - remote, remote);
    SyncArgs s2 = sd;
    s2.stamps = t.stamps;
    cudaError_t e = launch_gather_copy(pc, primary, st, &s2);
    t.end();
    if (e != cudaSuccess) return cuda_fail(e, "post-update gather kernel launch");
    clear_error();
    return HZ_OK;
  });
}

void p2p_release(hz_ctx* ctx) {
  auto& P = ctx->p2p;
  if (P.vw) {   // virtual world: pools are freed with the last context
    vw_release(ctx);
  } else if (P.pool) {
    // every rank must be done with every peer's pool before anyone unmaps / frees
    int* flag = nullptr;
    if (ctx->world_comm && cudaMalloc(&flag, sizeof(int)) == cudaSuccess) {
      ncclAllReduce(flag, flag, 1, ncclInt32, ncclSum, ctx->world_comm, nullptr);
      cudaStreamSynchronize(nullptr);
      cudaFree(flag);
    }
    for (int q = 0; q < ctx->world; ++q)
      if (q != ctx->rank && P.peer[q]) cudaIpcCloseMemHandle(P.peer[q]);
    cudaFree(P.pool);
  }
  if (P.abort_host) cudaFreeHost(P.abort_host);
  cudaGetLastError();
  P = hz_ctx::P2P{};
}

hz_status p2p_alloc_abort(hz_ctx* ctx) {
  auto& P = ctx->p2p;
  void* h = nullptr;
  P2P_CUDA(cudaHostAlloc(&h, 64, cudaHostAllocMapped | cudaHostAllocPortable), "abort word cudaHostAlloc");
  std::memset(h, 0, 64);
  void* d = nullptr;
  P2P_CUDA(cudaHostGetDevicePointer(&d, h, 0), "abort word cudaHostGetDevicePointer");
  P.abort_host = static_cast<unsigned*>(h);
  P.abort_dev = static_cast<unsigned*>(d);
  return HZ_OK;
}

}  // namespace hz

extern "C" {

hz_status hz_enable_p2p(hz_ctx* ctx, size_t pool_bytes) {
  using namespace hz;
  if (!ctx) return fail(HZ_ERR_INVALID, "ctx: NULL");
  if (ctx->p2p.on) return fail(HZ_ERR_INVALID, "ctx: P2P already enabled");
  if (ctx->world > kMaxWorld) return fail(HZ_ERR_UNSUPPORTED, "P2P transport supports at most 8 ranks");
  auto& P = ctx->p2p;
  const size_t total = align_up(kPoolHeader + pool_bytes, size_t(2) << 20);
  P2P_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  hz_status rc = p2p_alloc_abort(ctx);
  if (rc != HZ_OK) return rc;
  P2P_CUDA(cudaMalloc(&P.pool, total), "P2P pool cudaMalloc");
  P.bytes = total;
  P.used = kPoolHeader;
  P2P_CUDA(cudaMemset(P.pool, 0, kPoolHeader), "P2P pool header memset");
  cudaIpcMemHandle_t mine;
  P2P_CUDA(cudaIpcGetMemHandle(&mine, P.pool), "cudaIpcGetMemHandle");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  char* dev = nullptr;
  P2P_CUDA(cudaMalloc(&dev, 64 * ctx->world), "handle exchange cudaMalloc");
  P2P_CUDA(cudaMemcpy(dev + 64 * ctx->rank, &mine, 64, cudaMemcpyHostToDevice), "handle exchange copy");
  ncclResult_t r = ncclAllGather(dev + 64 * ctx->rank, dev, 64, ncclUint8, ctx->world_comm, nullptr);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather(IPC handles)");
  std::vector<cudaIpcMemHandle_t> all(ctx->world);
  P2P_CUDA(cudaMemcpy(all.data(), dev, 64 * ctx->world, cudaMemcpyDeviceToHost), "handle exchange copy back");
  cudaFree(dev);
  for (int q = 0; q < ctx->world; ++q) {
    if (q == ctx->rank) {
      P.peer[q] = P.pool;
      continue;
    }
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, all[q], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      p2p_release(ctx);
      return fail(HZ_ERR_UNSUPPORTED, std::string("cudaIpcOpenMemHandle (peer not reachable over P2P): ") +
                                          cudaGetErrorString(e));
    }
    P.peer[q] = static_cast<char*>(ptr);
  }
  // nobody starts using the pools before every rank has mapped every peer
  int* flag = nullptr;
  P2P_CUDA(cudaMalloc(&flag, sizeof(int)), "barrier cudaMalloc");
  r = ncclAllReduce(flag, flag, 1, ncclInt32, ncclSum, ctx->world_comm, nullptr);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce(barrier)");
  P2P_CUDA(cudaStreamSynchronize(nullptr), "barrier sync");
  cudaFree(flag);
  P.on = true;
  clear_error();
  return HZ_OK;
}

hz_status hz_p2p_enabled(const hz_ctx* ctx, int* out) {
  using namespace hz;
  if (!ctx || !out) return fail(HZ_ERR_INVALID, "ctx/out: NULL");
  *out = ctx->p2p.on ? 1 : 0;
  clear_error();
  return HZ_OK;
}

hz_status hz_set_wait_timeout(hz_ctx* ctx, double seconds) {
  using namespace hz;
  if (!ctx) return fail(HZ_ERR_INVALID, "ctx: NULL");
  if (!(seconds > 0.0) || seconds > 1e7) return fail(HZ_ERR_INVALID, "seconds: must be in (0, 1e7]");
  ctx->p2p.timeout_ns = static_cast<unsigned long long>(seconds * 1e9);
  clear_error();
  return HZ_OK;
}

hz_status hz_abort(hz_ctx* ctx) {
  using namespace hz;
  if (!ctx) return fail(HZ_ERR_INVALID, "ctx: NULL");
  if (ctx->p2p.abort_host) *reinterpret_cast<volatile unsigned*>(ctx->p2p.abort_host) = 2u;
  if (ctx->p2p.vw) vw_abort(ctx);
  clear_error();
  return HZ_OK;
}

hz_status hz_check(const hz_ctx* ctx) {
  using namespace hz;
  if (!ctx) return fail(HZ_ERR_INVALID, "ctx: NULL");
  hz_status rc = p2p_check(ctx);
  if (rc != HZ_OK) return rc;
  rc = check_async(ctx);
  if (rc != HZ_OK) return rc;
  clear_error();
  return HZ_OK;
}

hz_status hz_nvlink_probe(hz_ctx* ctx, int peer, size_t bytes, int reps, float* ms_out, void* stream) {
  using namespace hz;
  if (!ctx || !ms_out) return fail(HZ_ERR_INVALID, "ctx/ms_out: NULL");
  if (!ctx->p2p.on) return fail(HZ_ERR_INVALID, "ctx: P2P not enabled");
  if (peer < 0 || peer >= ctx->world) return fail(HZ_ERR_INVALID, "peer: must be in [0, world)");
  if (reps < 1) return fail(HZ_ERR_INVALID, "reps: must be >= 1");
  auto& P = ctx->p2p;
  if (bytes < 16 || bytes % 16 || kPoolHeader + bytes > P.bytes)
    return fail(HZ_ERR_INVALID, "bytes: must be a positive multiple of 16 within the pool");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned* sink = nullptr;
  cudaEvent_t a = nullptr, b = nullptr;
  P2P_CUDA(cudaMalloc(&sink, 4 * 4096), "probe sink cudaMalloc");
  P2P_CUDA(cudaMemsetAsync(sink, 0, 4 * 4096, st), "probe sink memset");
  P2P_CUDA(cudaEventCreate(&a), "probe event");
  P2P_CUDA(cudaEventCreate(&b), "probe event");
  const char* src = P.peer[peer] + kPoolHeader;
  P2P_CUDA(launch_peer_read(src, static_cast<int64_t>(bytes), sink, st), "probe warm-up launch");
  P2P_CUDA(cudaEventRecord(a, st), "probe event record");
  for (int i = 0; i < reps; ++i) P2P_CUDA(launch_peer_read(src, static_cast<int64_t>(bytes), sink, st), "probe launch");
  P2P_CUDA(cudaEventRecord(b, st), "probe event record");
  P2P_CUDA(cudaEventSynchronize(b), "probe sync");
  float ms = 0.f;
  P2P_CUDA(cudaEventElapsedTime(&ms, a, b), "probe elapsed");
  *ms_out = ms / reps;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  clear_error();
  return HZ_OK;
}

hz_status hz_flush(hz_ctx* ctx, void* stream) {
  using namespace hz;
  if (!ctx) return fail(HZ_ERR_INVALID, "ctx: NULL");
  if (!ctx->p2p.on) {
    clear_error();
    return HZ_OK;
  }
  hz_status rc = p2p_check(ctx);
  if (rc != HZ_OK) return rc;
  if ((rc = flush_prefetch(ctx, static_cast<cudaStream_t>(stream))) != HZ_OK) return rc;
  clear_error();
  return HZ_OK;
}

hz_status hz_p2p_capture_begin(hz_ctx* ctx) {
  using namespace hz;
  if (!ctx) return fail(HZ_ERR_INVALID, "ctx: NULL");
  if (!ctx->p2p.on) return fail(HZ_ERR_INVALID, "ctx: P2P not enabled");
  if (ctx->p2p.vw) return fail(HZ_ERR_UNSUPPORTED, "ctx: graph capture is not supported in a virtual world");
  if (ctx->p2p.capturing) return fail(HZ_ERR_INVALID, "ctx: capture already begun");
  if (ctx->p2p.pre_phase)
    return fail(HZ_ERR_INVALID, "ctx: a prefetched quantize (hz_allgather_params_next) is pending; gather that "
                                "layer before beginning a capture");
  if (ctx->p2p.pend.on)
    return fail(HZ_ERR_INVALID, "ctx: a deferred qgZ hop (hz_backward_step) is pending; call hz_flush (or finish "
                                "the backward pass) before beginning a capture");
  ctx->p2p.capturing = true;
  ctx->p2p.capture_start = ctx->p2p.phase;
  clear_error();
  return HZ_OK;
}

hz_status hz_p2p_capture_end(hz_ctx* ctx, void* stream, unsigned long long* span_out) {
  using namespace hz;
  if (!ctx) return fail(HZ_ERR_INVALID, "ctx: NULL");
  auto& P = ctx->p2p;
  if (!P.capturing) return fail(HZ_ERR_INVALID, "ctx: no capture in progress");
  hz_status rc = flush_prefetch(ctx, static_cast<cudaStream_t>(stream));   // inside the graph
  if (rc != HZ_OK) return rc;
  P.capturing = false;
  P.span = P.phase - P.capture_start;
  P.phase = P.capture_start;   // nothing captured has run yet
  cudaError_t e = launch_epoch_advance(reinterpret_cast<unsigned long long*>(P.pool + kEpochOff), P.span,
                                       static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "epoch-advance kernel launch");
  if (span_out) *span_out = P.span;
  clear_error();
  return HZ_OK;
}

hz_status hz_p2p_replayed(hz_ctx* ctx, unsigned long long n) {
  using namespace hz;
  if (!ctx) return fail(HZ_ERR_INVALID, "ctx: NULL");
  ctx->p2p.phase += n * ctx->p2p.span;
  ctx->p2p.epoch_host += n * ctx->p2p.span;
  clear_error();
  return HZ_OK;
}

hz_status hz_sym_alloc(hz_ctx* ctx, size_t bytes, void** out) {
  using namespace hz;
  if (!ctx || !out) return fail(HZ_ERR_INVALID, "ctx/out: NULL");
  if (!ctx->p2p.on) return fail(HZ_ERR_INVALID, "ctx: P2P not enabled (call hz_enable_p2p first)");
  size_t off = 0;
  hz_status rc = pool_alloc(ctx, bytes, &off);
  if (rc != HZ_OK) return rc;
  *out = ctx->p2p.pool + off;
  clear_error();
  return HZ_OK;
}

}  // extern "C"
