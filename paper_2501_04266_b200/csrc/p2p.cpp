// NVLink peer-memory transport (hz_enable_p2p): the per-level collectives are
// fused into the codec kernels instead of being staged through NCCL.
//
// Every rank owns one symmetric pool (cudaMalloc + cudaIpcGetMemHandle; the
// handles are exchanged with one ncclAllGather and opened with
// cudaIpcOpenMemHandle), so a buffer at pool offset X on this rank is at offset
// X in every peer's pool.  Allocations (hz_sym_alloc and the library's slots)
// are bump allocations made in the same order on every rank, hence symmetric.
//
// qwZ/hpZ all-gather (O7/O8): the owner quantizes its primary into a pool buffer
// (the caller's pool-allocated secondary when s == w); each rank then runs ONE
// gather+dequantize kernel whose pieces are the members' codes, read straight
// over NVLink — the gathered codes never land in HBM.  Backward: the same kernel
// over the members' secondaries.
// qgZ reduce-scatter (O9): level l's send buffer (quantize output, or the
// previous level's requantized sum) lives in the pool; the level-l reduce kernel
// reads chunk d_l of every group member's send buffer over NVLink and sums in
// ascending digit order — the all-to-all and the dequant+sum are one kernel.
//
// Ordering: every phase has a global number; producers wait until all ranks are
// done with the previous phase (no one still reads what they overwrite) and
// signal `ready`, consumers wait for `ready` and signal `done` (codec.cuh).
// All P2P calls of one context must be issued on one stream, in the same order
// on every rank (the NCCL discipline).
//
// Paired layers (hz_allgather_params_next / hz_backward_step): one dual kernel
// (k_gather_quantize) runs a gather of phase a and a quantize of phase a+1.  It waits
// for ready >= a (the gathered codes) and done >= a-1 (every rank finished every
// earlier phase, so nobody still reads what the quantize overwrites: the next layer's
// secondary, last read in an earlier backward phase, or the qgZ send slot, last read
// by the previous layer's reduce) and signals done = a and ready = a+1.  A prefetched
// quantize whose layer is not gathered next (another call comes first) leaves phase
// a+1 without a `done`; flush_prefetch completes it before the next phase starts.
#include <algorithm>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "ctx.h"

namespace hz {
int tune_param(const char* name, int dflt);
}

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

// pipelined-kernel chunk: about len / pk (HZ_TUNE pk, default 16) elements, a
// multiple of 1024 (4 blocks of 256), >= fchunk KiElements (default 64), and few
// enough chunks for the per-member flag arrays
int64_t chunk_elems(int64_t len) {
  int64_t c = (len + tune_param("pk", 16) - 1) / tune_param("pk", 16);
  const int64_t cap = (len + kMaxChunks - 1) / kMaxChunks;
  if (c < cap) c = cap;
  const int64_t lo = int64_t(tune_param("fchunk", 64)) * 1024;
  if (c < lo) c = lo;
  return (c + 1023) / 1024 * 1024;
}

template <typename T>
T* at(hz_ctx* ctx, int q, size_t off) {
  return reinterpret_cast<T*>(ctx->p2p.peer[q] + off);
}

size_t off_of(const hz_ctx* ctx, const void* local) {
  return static_cast<size_t>(static_cast<const char*>(local) - ctx->p2p.pool);
}

SyncArgs make_sync(hz_ctx* ctx, unsigned long long wait_ready, unsigned long long wait_done,
                   unsigned long long sig_ready, unsigned long long sig_done) {
  auto& P = ctx->p2p;
  SyncArgs s{};
  s.ready_local = reinterpret_cast<unsigned long long*>(P.pool + kReadyOff);
  s.done_local = reinterpret_cast<unsigned long long*>(P.pool + kDoneOff);
  for (int q = 0; q < ctx->world; ++q) {
    s.ready_remote[q] = reinterpret_cast<unsigned long long*>(P.peer[q] + kReadyOff) + ctx->rank;
    s.done_remote[q] = reinterpret_cast<unsigned long long*>(P.peer[q] + kDoneOff) + ctx->rank;
  }
  s.counter = reinterpret_cast<unsigned int*>(P.pool + kCounterOff);
  s.world = ctx->world;
  // thresholds are stored relative to the device epoch the kernel will see
  // (arguments: absolute phase numbers, 0 = none; phase numbers are > epoch_host)
  const unsigned long long e = P.epoch_host;
  s.en = (wait_ready ? kWaitReady : 0u) | (wait_done ? kWaitDone : 0u) | (sig_ready ? kSigReady : 0u) |
         (sig_done ? kSigDone : 0u);
  s.wait_ready = wait_ready - e;
  s.wait_done = wait_done - e;
  s.sig_ready = sig_ready - e;
  s.sig_done = sig_done - e;
  s.epoch = reinterpret_cast<const unsigned long long*>(P.pool + kEpochOff);
  s.mode = tune_param("p2p_sig", 1);   // fence.acq_rel.sys + relaxed.sys flag stores
  return s;
}

// Members of this rank's cumulative group of `level` (ranks that share every digit
// above `level`), as (off_level within range_0, rank), sorted by offset: piece k
// of the gathered layer is owned by the k-th entry.
std::vector<std::pair<int64_t, int>> cumulative_members(const hz_partition_t* p, int level) {
  int64_t stride[HZ_MAX_LEVELS];
  int64_t st = 1;
  for (int l = 0; l < p->levels; ++l) {
    stride[l] = st;
    st *= p->group[l];
  }
  int64_t base = p->rank;
  int64_t D = 1;
  for (int l = 0; l < level; ++l) {
    base -= p->digit[l] * stride[l];
    D *= p->group[l];
  }
  std::vector<std::pair<int64_t, int>> out;
  for (int64_t idx = 0; idx < D; ++idx) {
    int64_t rem = idx, r = base, off = 0;
    for (int l = 0; l < level; ++l) {
      const int d = static_cast<int>(rem % p->group[l]);
      rem /= p->group[l];
      r += d * stride[l];
      off += d * p->len[l + 1];
    }
    out.emplace_back(off, static_cast<int>(r));
  }
  std::sort(out.begin(), out.end());
  return out;
}

}  // namespace

// A prefetched quantize (hz_allgather_params_next) whose layer is not gathered next
// leaves its phase without a `done`; complete it before any other phase starts: a
// one-CTA kernel signalling done(pre_phase) — nobody reads those codes, and every
// earlier read of this rank is complete in stream order.
hz_status flush_prefetch(hz_ctx* ctx, cudaStream_t st) {
  auto& P = ctx->p2p;
  if (!P.pre_phase) return HZ_OK;
  const unsigned long long ph = P.pre_phase;
  P.pre_phase = 0;
  P.pre_codes = P.pre_primary = nullptr;
  Pieces pc{};
  pc.n = 1;
  SyncArgs s = make_sync(ctx, 0, 0, 0, ph);
  return run_gather_dequantize(pc, 0, 8, 256, nullptr, HZ_BF16, st, 0, &s, 0);
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
         tune_param("pushf", 0) == 0 && tune_param("fused", 0) == 0 && tune_param("nofuse", 0) == 0;
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
  // every call is a phase, even without peers to read from: it may write a
  // secondary that peers read in a later backward phase (s > w), and the final
  // kernel's done(phase) is what tells them the write (incl. its copies) is complete
  // this layer's primary already quantized by the previous call's dual kernel (the
  // prefetch of hz_allgather_params_next), in phase pre_phase, with no phase since
  const bool pre = !backward && s == w && P.pre_phase != 0 && P.pre_phase == P.phase &&
                   P.pre_codes == sec_codes && P.pre_primary == primary;
  if (pre) {
    P.pre_phase = 0;
    P.pre_codes = P.pre_primary = nullptr;
  } else if ((rc = flush_prefetch(ctx, st)) != HZ_OK) {
    return rc;
  }
  const unsigned long long phase = pre ? P.phase : ++P.phase;
  const int64_t plen = p->len[top];
  int me = 0;
  for (int k = 0; k < D; ++k)
    if (members[k].second == ctx->rank) me = k;
  // forward with s == w, hybrid push/pull (HZ_TUNE pushf = % of each piece pushed by
  // the quantize kernel, in whole 1024-element tiles).  Default 0 = pull only: on
  // B200 the pushes cost the quantize kernel about as much NVLink time as they save
  // the gather (profiles/push_pull_r01.md).
  int64_t push_lim = 0;
  if (!backward && s == w && D > 1 && B == 256)
    push_lim = plen * tune_param("pushf", 0) / 100 / 1024 * 1024;

  if (!backward && s == w && D > 1 && B == 256 && tune_param("fused", 0)) {
    // A2 + A3 + A5 in ONE kernel: quantize the own primary chunk by chunk into the
    // (peer-readable) secondary, publish each chunk, and dequantize every member's
    // chunks as they become ready — NVLink transfers overlap the quantization.
    FusedAGArgs h{};
    h.x = primary;
    h.dt = dt;
    h.bits = bits;
    h.qc = sec_codes;
    h.qs = sec_scales;
    h.D = D;
    h.plen = plen;
    h.C = chunk_elems(plen);
    h.nch = static_cast<int>((plen + h.C - 1) / h.C);
    int64_t remote = 0;
    for (int k = 0; k < D; ++k) {
      const int m = members[k].second;
      if (m == ctx->rank) h.me = k;
      h.pc[k] = at<const uint8_t>(ctx, m, off_of(ctx, sec_codes));
      h.ps[k] = at<const float>(ctx, m, off_of(ctx, sec_scales));
      if (m != ctx->rank) remote += code_bytes(plen, bits) + plen / B * 4;
    }
    for (int k = 0; k < D; ++k)
      h.flags_remote[k] = at<unsigned long long>(ctx, members[k].second, kChunkAGOff) + h.me * kMaxChunks;
    h.flags = at<unsigned long long>(ctx, ctx->rank, kChunkAGOff);
    h.work = at<unsigned long long>(ctx, ctx->rank, kWorkAGOff);
    h.cnt = at<unsigned int>(ctx, ctx->rank, kCntAGOff);
    h.y = full_out;
    h.out_dt = out_dt;
    h.phase = phase - P.epoch_host;
    h.epoch = at<const unsigned long long>(ctx, ctx->rank, kEpochOff);
    SyncArgs sy = make_sync(ctx, 0, phase - 1, 0, phase);
    const int64_t local = p->len[w] * elem_bytes(dt) + code_bytes(plen, bits) + plen / B * 4 +
                          code_bytes(Np, bits) + Np / B * 4 - remote + Np * elem_bytes(out_dt);
    static int dbg_calls = 0;
    const bool dbg = tune_param("pdbg", 0) && ++dbg_calls == tune_param("pdbg", 0);
    if (dbg) {   // diagnostic timeline of one call (HZ_TUNE pdbg=<call number>), printed to stderr
      h.dbg = at<unsigned long long>(ctx, ctx->rank, kDbgOff);
      std::vector<unsigned long long> init(size_t(kMaxChunks) * 4, 0ull);
      for (int c = 0; c < h.nch; ++c) init[c * 4 + 1] = ~0ull;
      cudaMemcpyAsync(h.dbg, init.data(), init.size() * 8, cudaMemcpyHostToDevice, st);
      cudaStreamSynchronize(st);
    }
    TraceScope t(st, "ag_fused", w, bits, Np, local, remote);
    sy.stamps = t.stamps;
    cudaError_t e = launch_ag_fused(h, st, sy);
    t.end();
    if (e != cudaSuccess) return cuda_fail(e, "fused all-gather kernel launch");
    if (dbg) {
      std::vector<unsigned long long> tl(size_t(kMaxChunks) * 4);
      cudaStreamSynchronize(st);
      cudaMemcpy(tl.data(), h.dbg, tl.size() * 8, cudaMemcpyDeviceToHost);
      const unsigned long long t0 = tl[(kMaxChunks - 1) * 4];
      fprintf(stderr, "[hz pdbg rank %d] ag_pipe plen=%lld C=%lld nch=%d (us from entry: last-arrive publish "
              "first-consumer-start last-consumer-end)\n", ctx->rank, (long long)plen, (long long)h.C, h.nch);
      for (int c = 0; c < h.nch; ++c)
        fprintf(stderr, "  c=%3d %8.2f %8.2f %8.2f %8.2f\n", c, (tl[c * 4 + 3] - t0) * 1e-3, (tl[c * 4] - t0) * 1e-3,
                (tl[c * 4 + 1] - t0) * 1e-3, (tl[c * 4 + 2] - t0) * 1e-3);
    }
    clear_error();
    return HZ_OK;
  }
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
    SyncArgs sq = make_sync(ctx, 0, phase - 1, phase, 0);
    if (push_lim > 0) {
      // hybrid push/pull: the quantize kernel (HBM-bound, NVLink idle) also stores
      // the first push_lim codes of its piece into every member's receive buffer;
      // the gather below pulls only the rest over NVLink
      if ((rc = slot(ctx, P.ag_recv_c, code_bytes(D * plen, 8))) != HZ_OK) return rc;
      if ((rc = slot(ctx, P.ag_recv_s, D * plen / B * 4)) != HZ_OK) return rc;
      PushDst dst{};
      int64_t pushed = 0;
      for (int k = 0; k < D; ++k) {
        if (members[k].second == ctx->rank) continue;
        dst.c[dst.n] = at<uint8_t>(ctx, members[k].second, P.ag_recv_c.off) + code_bytes(me * plen, bits);
        dst.s[dst.n] = at<float>(ctx, members[k].second, P.ag_recv_s.off) + me * plen / B;
        ++dst.n;
        pushed += code_bytes(push_lim, bits) + push_lim / B * 4;
      }
      dst.lim = push_lim;
      if ((rc = run_quantize_push(primary, dt, plen, bits, qc, qs, nullptr, out_dt, dst, st, w, &sq, pushed)) !=
          HZ_OK)
        return rc;
    } else if (!pre && (rc = run_quantize(primary, dt, p->len[w], bits, B, qc, qs, st, w, &sq)) != HZ_OK) {
      return rc;
    }
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
    if (m == ctx->rank) continue;
    remote += code_bytes(plen - push_lim, bits) + (plen - push_lim) / B * 4;
    if (push_lim > 0) {   // the pushed head of piece k is already in the local receive buffer
      pc.cr[k] = at<const uint8_t>(ctx, ctx->rank, P.ag_recv_c.off) + code_bytes(k * plen, bits);
      pc.sr[k] = at<const float>(ctx, ctx->rank, P.ag_recv_s.off) + k * plen / B;
    }
  }
  pc.split = push_lim;
  if (!backward && s < w) {   // A4, s < w: keep range_s of the gathered codes
    pc.sec_c = sec_codes;
    pc.sec_s = sec_scales;
    pc.sec_lo = p->off[s];
    pc.sec_hi = p->off[s] + len_s;
  }
  if (!backward && next && next->codes != sec_codes && next->scales != sec_scales &&
      p2p_next_fusable(ctx, p, bits, out_dt, *next)) {
    // gather this layer (phase) || quantize the next layer's primary (phase + 1) in one
    // launch.  Waits: the members' codes of this phase are ready, and every rank is
    // done with every phase before it (nobody still reads the next layer's secondary,
    // last read in an earlier backward phase).  Signals done(phase), ready(phase + 1).
    const unsigned long long nph = ++P.phase;
    const hz_partition_t* q = next->p;
    SyncArgs sd = make_sync(ctx, phase, phase - 1, nph, phase);
    if ((rc = run_gather_quantize(pc, Np, bits, full_out, out_dt, next->primary, dt, q->len[q->w], bits, next->codes,
                                  next->scales, st, sd, remote)) != HZ_OK)
      return rc;
    P.pre_phase = nph;
    P.pre_codes = next->codes;
    P.pre_primary = next->primary;
    clear_error();
    return HZ_OK;
  }
  SyncArgs sd = backward ? make_sync(ctx, 0, phase - 1, 0, phase) : make_sync(ctx, phase, 0, 0, phase);
  if ((rc = run_gather_dequantize(pc, Np, bits, B, full_out, out_dt, st, 0, &sd, remote)) != HZ_OK)
    return rc;
  clear_error();
  return HZ_OK;
}

// qgZ over NVLink, push mode: every producer (the level-`from` quantize, each
// level's requantizing reduce) stores the chunk destined to member j straight into
// member j's level receive buffer, at the producer's own digit; every reduce then
// reads its g inputs from local HBM (ascending digit = the oracle's summation order).
hz_status p2p_reduce_scatter_push(hz_ctx* ctx, const hz_partition_t* p, const void* grad, hz_dtype dt,
                                  int from_level, int to_level, const int* bits_per_level, float* shard,
                                  int accumulate, cudaStream_t st) {
  auto& P = ctx->p2p;
  const int B = p->block;
  hz_status rc;
  for (int l = from_level; l <= to_level; ++l) {   // level-l receive buffers (8-bit capacity)
    if ((rc = slot(ctx, P.rs_recv_c[l], code_bytes(p->len[l - 1], 8))) != HZ_OK) return rc;
    if ((rc = slot(ctx, P.rs_recv_s[l], p->len[l - 1] / B * 4)) != HZ_OK) return rc;
  }
  int64_t stride[HZ_MAX_LEVELS];
  int64_t sacc = 1;
  for (int l = 0; l < p->levels; ++l) {
    stride[l] = sacc;
    sacc *= p->group[l];
  }
  // destinations of level l's chunks: member j gets chunk j at this rank's digit
  auto dest_of = [&](int l, int bits, PushDst& dst, int64_t& remote) {
    const int g = p->group[l - 1];
    const int d = p->digit[l - 1];
    const int64_t cl = p->len[l];
    dst = PushDst{};
    dst.n = g;
    dst.scatter = 1;
    dst.seg = cl;
    remote = 0;
    for (int j = 0; j < g; ++j) {
      const int m = static_cast<int>(p->rank + (static_cast<int64_t>(j) - d) * stride[l - 1]);
      dst.c[j] = at<uint8_t>(ctx, m, P.rs_recv_c[l].off) + code_bytes(d * cl, bits);
      dst.s[j] = at<float>(ctx, m, P.rs_recv_s[l].off) + d * cl / B;
      if (m != ctx->rank) remote += code_bytes(cl, bits) + cl / B * 4;
    }
  };
  const unsigned long long base = P.phase;
  P.phase += static_cast<unsigned long long>(to_level - from_level + 1);
  auto phase_of = [&](int l) { return base + static_cast<unsigned long long>(l - from_level + 1); };
  {   // A7 + A8: quantize range_{from-1} and push chunk j to member j
    const int l = from_level;
    PushDst dst;
    int64_t remote;
    dest_of(l, bits_per_level[l - 1], dst, remote);
    const unsigned long long ph = phase_of(l);
    SyncArgs sq = make_sync(ctx, 0, ph - 1, ph, 0);
    if ((rc = run_quantize_push(grad, dt, p->len[l - 1], bits_per_level[l - 1], nullptr, nullptr, nullptr, HZ_F32, dst,
                                st, l, &sq, remote)) != HZ_OK)
      return rc;
  }
  for (int l = from_level; l <= to_level; ++l) {   // A9 (+ A8 of the next level) / A10
    const int g = p->group[l - 1];
    const int bits = bits_per_level[l - 1];
    const int64_t cl = p->len[l];
    const uint8_t* ptr_c[kMaxG];
    const float* ptr_s[kMaxG];
    for (int j = 0; j < g; ++j) {
      ptr_c[j] = at<const uint8_t>(ctx, ctx->rank, P.rs_recv_c[l].off) + code_bytes(j * cl, bits);
      ptr_s[j] = at<const float>(ctx, ctx->rank, P.rs_recv_s[l].off) + j * cl / B;
    }
    const unsigned long long ph = phase_of(l);
    if (l < to_level) {
      PushDst dst;
      int64_t remote;
      dest_of(l + 1, bits_per_level[l], dst, remote);
      SyncArgs sr = make_sync(ctx, ph, ph - 1, ph + 1, ph);
      if ((rc = run_reduce_push(g, ptr_c, ptr_s, cl, bits, bits_per_level[l], dst, st, l, &sr, remote)) != HZ_OK)
        return rc;
    } else {
      SyncArgs sr = make_sync(ctx, ph, 0, 0, ph);
      if ((rc = run_reduce(g, ptr_c, ptr_s, cl, bits, B, 0, nullptr, nullptr, shard, accumulate, st, l, &sr, 0)) !=
          HZ_OK)
        return rc;
    }
  }
  clear_error();
  return HZ_OK;
}

bool p2p_prev_fusable(const hz_ctx* ctx, const hz_partition_t* p, int from_level, const PrevG& pg) {
  const hz_partition_t* q = pg.p;
  return ctx->p2p.on && q && p->block == 256 && q->block == 256 && p->len[from_level - 1] > 0 &&
         gather_quantize_supported(256, pg.bits, pg.out_dt) &&
         in_pool(ctx, pg.sec_codes, code_bytes(q->len[q->s], pg.bits)) &&
         in_pool(ctx, pg.sec_scales, q->len[q->s] / 256 * 4) && static_cast<int>(cumulative_members(q, q->s).size()) <=
                                                                   kMaxWorld &&
         tune_param("rspush", 0) == 0 && tune_param("fused", 0) == 0 && tune_param("nofuse", 0) == 0;
}

hz_status p2p_reduce_scatter(hz_ctx* ctx, const hz_partition_t* p, const void* grad, hz_dtype dt,
                             int from_level, int to_level, const int* bits_per_level, float* shard,
                             int accumulate, cudaStream_t st, const PrevG* prev) {
  auto& P = ctx->p2p;
  const int B = p->block;
  hz_status rc;
  if ((rc = flush_prefetch(ctx, st)) != HZ_OK) return rc;
  // the previous layer's backward gather (phase gph) fused into this call's first
  // quantize (hz_backward_step; the caller checked p2p_prev_fusable)
  unsigned long long gph = 0;
  Pieces gpc{};
  int64_t gremote = 0;
  if (prev) {
    gph = ++P.phase;
    const hz_partition_t* q = prev->p;
    const auto members = cumulative_members(q, q->s);
    gpc.n = static_cast<int>(members.size());
    gpc.len = q->len[q->s];
    for (int k = 0; k < gpc.n; ++k) {
      const int m = members[k].second;
      gpc.c[k] = at<const uint8_t>(ctx, m, off_of(ctx, prev->sec_codes));
      gpc.s[k] = at<const float>(ctx, m, off_of(ctx, prev->sec_scales));
      if (m != ctx->rank) gremote += code_bytes(gpc.len, prev->bits) + gpc.len / 256 * 4;
    }
  }
  // full push for qgZ measured slower than pull on B200: HZ_TUNE rspush=1
  bool push = B == 256 && tune_param("rspush", 0) && !tune_param("fused", 0);
  for (int l = from_level; l < to_level; ++l) push = push && push_reduce_supported(p->group[l - 1], B);
  for (int l = from_level; l <= to_level; ++l)
    if (p->group[l - 1] > kMaxG) return fail(HZ_ERR_UNSUPPORTED, "group size > 16 at one level");
  if (push) return p2p_reduce_scatter_push(ctx, p, grad, dt, from_level, to_level, bits_per_level, shard, accumulate,
                                           st);
  for (int l = from_level; l <= to_level; ++l) {   // level-l send buffers (8-bit capacity)
    if ((rc = slot(ctx, P.rs_c[l], code_bytes(p->len[l - 1], 8))) != HZ_OK) return rc;
    if ((rc = slot(ctx, P.rs_s[l], p->len[l - 1] / B * 4)) != HZ_OK) return rc;
  }
  int64_t stride[HZ_MAX_LEVELS];
  int64_t sacc = 1;
  for (int l = 0; l < p->levels; ++l) {
    stride[l] = sacc;
    sacc *= p->group[l];
  }
  const unsigned long long base = P.phase;
  P.phase += static_cast<unsigned long long>(to_level - from_level + 1);
  auto phase_of = [&](int l) { return base + static_cast<unsigned long long>(l - from_level + 1); };

  int first = from_level;   // first level handled by the per-level kernels below
  if (B == 256 && fused_rs_supported(p->group[from_level - 1]) && tune_param("fused", 0)) {
    // A7 + A8 + A9 of the first level in ONE kernel: quantize the own input chunk by
    // chunk (destinations interleaved), publish each chunk to its destination, and
    // reduce the members' chunks destined here as they become ready.
    const int l = from_level;
    const int g = p->group[l - 1];
    const int d = p->digit[l - 1];
    const int bits = bits_per_level[l - 1];
    const int64_t cl = p->len[l];
    const unsigned long long ph = phase_of(l);
    FusedRSArgs h{};
    h.x = grad;
    h.dt = dt;
    h.bits_in = bits;
    h.bits_out = l < to_level ? bits_per_level[l] : 0;
    h.acc = l < to_level ? 0 : accumulate;
    h.qc = at<uint8_t>(ctx, ctx->rank, P.rs_c[l].off);
    h.qs = at<float>(ctx, ctx->rank, P.rs_s[l].off);
    h.g = g;
    h.d = d;
    h.cl = cl;
    h.C = chunk_elems(cl);
    h.ncl = static_cast<int>((cl + h.C - 1) / h.C);
    for (int j = 0; j < g; ++j) {
      const int m = static_cast<int>(p->rank + (static_cast<int64_t>(j) - d) * stride[l - 1]);
      h.mc[j] = at<const uint8_t>(ctx, m, P.rs_c[l].off) + code_bytes(d * cl, bits);
      h.ms[j] = at<const float>(ctx, m, P.rs_s[l].off) + d * cl / B;
      h.flags_remote[j] = at<unsigned long long>(ctx, m, kChunkRSOff) + d * kMaxChunks;
    }
    h.flags = at<unsigned long long>(ctx, ctx->rank, kChunkRSOff);
    h.work = at<unsigned long long>(ctx, ctx->rank, kWorkRSOff);
    h.cnt = at<unsigned int>(ctx, ctx->rank, kCntRSOff);
    h.of = shard;
    if (l < to_level) {
      h.oc = at<uint8_t>(ctx, ctx->rank, P.rs_c[l + 1].off);
      h.os = at<float>(ctx, ctx->rank, P.rs_s[l + 1].off);
    }
    h.phase = ph - P.epoch_host;
    h.epoch = at<const unsigned long long>(ctx, ctx->rank, kEpochOff);
    SyncArgs sy = l < to_level ? make_sync(ctx, 0, ph - 1, ph + 1, ph) : make_sync(ctx, 0, ph - 1, 0, ph);
    const int64_t n_in = p->len[l - 1];
    const int64_t remote = (g - 1) * (code_bytes(cl, bits) + cl / B * 4);
    const int64_t out = h.bits_out ? code_bytes(cl, h.bits_out) + cl / B * 4 : cl * 4 * (h.acc ? 2 : 1);
    const int64_t local = n_in * elem_bytes(dt) + code_bytes(n_in, bits) + n_in / B * 4 +
                          g * (code_bytes(cl, bits) + cl / B * 4) - remote + out;
    TraceScope t(st, "rs_fused", l, bits, n_in, local, remote);
    sy.stamps = t.stamps;
    cudaError_t e = launch_rs_fused(h, st, sy);
    t.end();
    if (e != cudaSuccess) return cuda_fail(e, "fused reduce-scatter kernel launch");
    first = l + 1;
  } else if (prev) {
    // previous layer's backward gather (phase gph) || A7 of this layer (phase gph + 1):
    // waits until every rank is done with every phase before gph (the secondaries
    // are complete, nobody reads the send buffer any more); signals done(gph) and
    // ready(gph + 1) for the level-`from` reduce below
    const unsigned long long ph = phase_of(from_level);
    SyncArgs sq = make_sync(ctx, 0, gph - 1, ph, gph);
    if ((rc = run_gather_quantize(gpc, prev->p->padded_numel, prev->bits, prev->full_out, prev->out_dt, grad, dt,
                                  p->len[from_level - 1], bits_per_level[from_level - 1],
                                  at<uint8_t>(ctx, ctx->rank, P.rs_c[from_level].off),
                                  at<float>(ctx, ctx->rank, P.rs_s[from_level].off), st, sq, gremote)) != HZ_OK)
      return rc;
  } else {
    // A7: quantize the input range_{from-1} into this rank's level-`from` send buffer
    const unsigned long long ph = phase_of(from_level);
    SyncArgs sq = make_sync(ctx, 0, ph - 1, ph, 0);
    if ((rc = run_quantize(grad, dt, p->len[from_level - 1], bits_per_level[from_level - 1], B,
                           at<uint8_t>(ctx, ctx->rank, P.rs_c[from_level].off),
                           at<float>(ctx, ctx->rank, P.rs_s[from_level].off), st, from_level, &sq)) != HZ_OK)
      return rc;
  }
  for (int l = first; l <= to_level; ++l) {
    const int g = p->group[l - 1];
    const int d = p->digit[l - 1];
    const int bits = bits_per_level[l - 1];
    const int64_t cl = p->len[l];
    if (g > kMaxG) return fail(HZ_ERR_UNSUPPORTED, "group size > 16 at one level");
    const uint8_t* ptr_c[kMaxG];
    const float* ptr_s[kMaxG];
    for (int j = 0; j < g; ++j) {   // A8+A9: chunk d of member j's send buffer, over NVLink
      const int m = static_cast<int>(p->rank + (static_cast<int64_t>(j) - d) * stride[l - 1]);
      ptr_c[j] = at<const uint8_t>(ctx, m, P.rs_c[l].off) + code_bytes(d * cl, bits);
      ptr_s[j] = at<const float>(ctx, m, P.rs_s[l].off) + d * cl / B;
    }
    const unsigned long long ph = phase_of(l);
    const int64_t remote = (g - 1) * (code_bytes(cl, bits) + cl / B * 4);
    if (l < to_level) {
      SyncArgs sr = make_sync(ctx, ph, ph - 1, ph + 1, ph);
      if ((rc = run_reduce(g, ptr_c, ptr_s, cl, bits, B, bits_per_level[l],
                           at<uint8_t>(ctx, ctx->rank, P.rs_c[l + 1].off),
                           at<float>(ctx, ctx->rank, P.rs_s[l + 1].off), nullptr, 0, st, l, &sr, remote)) != HZ_OK)
        return rc;
    } else {
      SyncArgs sr = make_sync(ctx, ph, 0, 0, ph);
      if ((rc = run_reduce(g, ptr_c, ptr_s, cl, bits, B, 0, nullptr, nullptr, shard, accumulate, st, l, &sr, remote)) !=
          HZ_OK)
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
  int64_t stride[HZ_MAX_LEVELS];
  int64_t sacc = 1;
  for (int l = 0; l < p->levels; ++l) {
    stride[l] = sacc;
    sacc *= p->group[l];
  }
  const size_t off[2] = {P.ar_a.off, P.ar_b.off};
  const unsigned long long base = P.phase;
  P.phase += static_cast<unsigned long long>(to_level - from_level + 1);
  // copy-in (producer of phase base+1): the slot may still be read in phase base
  {
    Pieces pc{};
    pc.n = 1;
    pc.len = n;
    pc.c[0] = reinterpret_cast<const uint8_t*>(in);
    SyncArgs sq = make_sync(ctx, 0, base, base + 1, 0);
    if ((rc = run_sum(pc, n, at<float>(ctx, ctx->rank, off[0]), st, from_level, &sq, 0)) != HZ_OK) return rc;
  }
  int cur = 0;
  for (int l = from_level; l <= to_level; ++l) {
    const int g = p->group[l - 1];
    const int d = p->digit[l - 1];
    const unsigned long long ph = base + static_cast<unsigned long long>(l - from_level + 1);
    Pieces pc{};
    pc.n = g;
    pc.len = n;
    int64_t remote = 0;
    for (int j = 0; j < g; ++j) {
      const int m = static_cast<int>(p->rank + (static_cast<int64_t>(j) - d) * stride[l - 1]);
      pc.c[j] = at<const uint8_t>(ctx, m, off[cur]);
      if (m != ctx->rank) remote += n * 4;
    }
    SyncArgs sr = l < to_level ? make_sync(ctx, ph, ph - 1, ph + 1, ph) : make_sync(ctx, ph, ph - 1, 0, ph);
    if ((rc = run_sum(pc, n, at<float>(ctx, ctx->rank, off[cur ^ 1]), st, l, &sr, remote)) != HZ_OK) return rc;
    cur ^= 1;
  }
  // select range_to (local; the slot's next writer waits for this rank's done flag,
  // which follows this copy in stream order)
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
  const unsigned long long phase = ++P.phase;
  char* mine = at<char>(ctx, ctx->rank, P.upd.off);
  SyncArgs sq = make_sync(ctx, 0, phase - 1, phase, 0);
  if ((rc = run_adamw(g, th, m, v, mine, dt, lenL, hp, st, &sq)) != HZ_OK) return rc;
  // members: vary digits w+1..L, keep digits 1..w
  int64_t stride[HZ_MAX_LEVELS];
  int64_t sacc = 1;
  for (int l = 0; l < L; ++l) {
    stride[l] = sacc;
    sacc *= p->group[l];
  }
  int64_t base = p->rank, D = 1;
  for (int l = w; l < L; ++l) {
    base -= p->digit[l] * stride[l];
    D *= p->group[l];
  }
  if (D > kMaxWorld) return fail(HZ_ERR_UNSUPPORTED, "P2P gather over more than 8 ranks");
  std::vector<std::pair<int64_t, int>> mem;
  for (int64_t idx = 0; idx < D; ++idx) {
    int64_t rem = idx, r = base, off = 0;
    for (int l = w; l < L; ++l) {
      const int d = static_cast<int>(rem % p->group[l]);
      rem /= p->group[l];
      r += d * stride[l];
      off += d * p->len[l + 1];
    }
    mem.emplace_back(off, static_cast<int>(r));
  }
  std::sort(mem.begin(), mem.end());
  Pieces pc{};
  pc.n = static_cast<int>(D);
  pc.len = lenL * eb;   // bytes
  int64_t remote = 0;
  for (int k = 0; k < pc.n; ++k) {
    pc.c[k] = at<const uint8_t>(ctx, mem[k].second, P.upd.off);
    if (mem[k].second != ctx->rank) remote += pc.len;
  }
  SyncArgs sd = make_sync(ctx, phase, 0, 0, phase);
  TraceScope t(st, "gather_copy", w, 16, lenL * D, D * pc.len * 2 - remote, remote);
  sd.stamps = t.stamps;
  cudaError_t e = launch_gather_copy(pc, primary, st, &sd);
  t.end();
  if (e != cudaSuccess) return cuda_fail(e, "post-update gather kernel launch");
  clear_error();
  return HZ_OK;
}

void p2p_release(hz_ctx* ctx) {
  auto& P = ctx->p2p;
  if (!P.pool) return;
  // every rank must be done with every peer's pool before anyone unmaps / frees
  int* flag = nullptr;
  if (cudaMalloc(&flag, sizeof(int)) == cudaSuccess) {
    ncclAllReduce(flag, flag, 1, ncclInt32, ncclSum, ctx->world_comm, nullptr);
    cudaStreamSynchronize(nullptr);
    cudaFree(flag);
  }
  for (int q = 0; q < ctx->world; ++q)
    if (q != ctx->rank && P.peer[q]) cudaIpcCloseMemHandle(P.peer[q]);
  cudaFree(P.pool);
  cudaGetLastError();
  P = hz_ctx::P2P{};
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

hz_status hz_p2p_capture_begin(hz_ctx* ctx) {
  using namespace hz;
  if (!ctx) return fail(HZ_ERR_INVALID, "ctx: NULL");
  if (!ctx->p2p.on) return fail(HZ_ERR_INVALID, "ctx: P2P not enabled");
  if (ctx->p2p.capturing) return fail(HZ_ERR_INVALID, "ctx: capture already begun");
  if (ctx->p2p.pre_phase)
    return fail(HZ_ERR_INVALID, "ctx: a prefetched quantize (hz_allgather_params_next) is pending; gather that "
                                "layer before beginning a capture");
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
