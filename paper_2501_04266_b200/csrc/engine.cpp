// Level engine: NCCL communicators per hierarchy level and the two collectives of
// the hot path, stream-ordered on the caller's stream.
//
//   hz_allgather_params     qwZ + hpZ (O7/O8): Table VII
//   hz_reduce_scatter_grads qgZ (O9):          P:122, Table VIII
//   hz_flat_*               the ZeRO-3 baseline rows of Tables VII/VIII
//
// Communicators: one world communicator plus, for every level l with g_l > 1,
// ncclCommSplit(world, color = rank - d_l*stride_l, key = d_l): the level-l
// exchange group, whose communicator rank equals the level digit d_l.  On one
// NVSwitch box every level runs over NVLink at the same per-GPU bandwidth; the
// hierarchy saves bytes ((g_l-1)/g_l of a shrinking range per level) and peers.
//
// All-gather: codes and scales live in two SoA arrays indexed by global element
// / block, so the level-l gather concatenating the group's range_l pieces into
// range_{l-1} is an in-place ncclAllGather on both arrays (one NCCL group).
// Reduce-scatter: the level-l send buffer is the SoA code of range_{l-1}; chunk j
// (= destination digit j) is a contiguous slice of both arrays, so the
// all-to-all is grouped ncclSend/ncclRecv of slices; the own chunk is read in
// place by the reduce kernel and never enters NCCL.
#include <cmath>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "ctx.h"

namespace hz {

int tune_param(const char* name, int dflt);

hz_status cuda_fail(cudaError_t e, const char* what) {
  return fail(HZ_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

hz_status nccl_fail(ncclResult_t r, const char* what) {
  return fail(HZ_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

#define HZ_NCCL(call, what)                     \
  do {                                          \
    ncclResult_t r_ = (call);                   \
    if (r_ != ncclSuccess) return nccl_fail(r_, what); \
  } while (0)

#define HZ_CUDA(call, what)                     \
  do {                                          \
    cudaError_t e_ = (call);                    \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

hz_status grow(hz_ctx::Buf& b, size_t need) {
  if (need <= b.cap) return HZ_OK;
  const size_t gran = size_t(2) << 20;
  const size_t cap = (need + gran - 1) / gran * gran;
  if (b.p) {
    HZ_CUDA(cudaDeviceSynchronize(), "workspace growth: cudaDeviceSynchronize");
    HZ_CUDA(cudaFree(b.p), "workspace growth: cudaFree");
    b.p = nullptr;
    b.cap = 0;
  }
  HZ_CUDA(cudaMalloc(&b.p, cap), "workspace growth: cudaMalloc");
  b.cap = cap;
  return HZ_OK;
}

namespace {
void free_buf(hz_ctx::Buf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
}

}  // namespace

// Asynchronous NCCL errors of ANY communicator of the context (world, levels, merged
// hops: the level communicators carry the traffic) and the P2P abort word.  On an
// NCCL error every communicator is aborted (ncclCommAbort: no later call can hang on
// a dead peer) and every later call reports HZ_ERR_NCCL.
hz_status check_async(const hz_ctx* ctx) {
  hz_status rc = p2p_check(ctx);
  if (rc != HZ_OK) return rc;
  hz_ctx* c = const_cast<hz_ctx*>(ctx);
  if (c->nccl_dead) return fail(HZ_ERR_NCCL, "NCCL communicators were aborted after an asynchronous error: " + c->nccl_err);
  std::vector<ncclComm_t*> comms;
  if (c->world_comm) comms.push_back(&c->world_comm);
  for (auto& x : c->lvl)
    if (x) comms.push_back(&x);
  for (auto& row : c->hop_comm)
    for (auto& x : row)
      if (x) comms.push_back(&x);
  for (ncclComm_t* cm : comms) {
    ncclResult_t r = ncclSuccess;
    if (ncclCommGetAsyncError(*cm, &r) == ncclSuccess && r != ncclSuccess && r != ncclInProgress) {
      c->nccl_err = ncclGetErrorString(r);
      for (ncclComm_t* k : comms) {
        ncclCommAbort(*k);
        *k = nullptr;
      }
      c->nccl_dead = true;
      return fail(HZ_ERR_NCCL, "asynchronous NCCL error from an earlier call (communicators aborted): " + c->nccl_err);
    }
  }
  return HZ_OK;
}

// Communicator of the merged hop over levels a..b (a == b: the level communicator),
// split from the world communicator on first use — a collective call, made by every
// rank at the same point of the same call sequence.  Comm rank = merged digit.
hz_status hop_comm(hz_ctx* ctx, int a, int b, ncclComm_t* out) {
  if (a == b) {
    *out = ctx->lvl[a - 1];
    return HZ_OK;
  }
  ncclComm_t& c = ctx->hop_comm[a - 1][b - 1];
  if (!c) {
    int stride = 1, color = ctx->rank, key = 0, kstride = 1;
    for (int l = 1; l <= ctx->levels; ++l) {
      if (l >= a && l <= b) {
        color -= ctx->digit[l - 1] * stride;
        key += ctx->digit[l - 1] * kstride;
        kstride *= ctx->group[l - 1];
      }
      stride *= ctx->group[l - 1];
    }
    ncclResult_t r = ncclCommSplit(ctx->world_comm, color, key, &c, nullptr);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommSplit(merged hop)");
  }
  *out = c;
  return HZ_OK;
}

hz_status check_partition(const hz_ctx* ctx, const hz_partition_t* p) {
  if (!ctx) return fail(HZ_ERR_INVALID, "ctx: NULL");
  if (!p) return fail(HZ_ERR_INVALID, "p: NULL");
  if (p->rank != ctx->rank || p->world != ctx->world || p->levels != ctx->levels)
    return fail(HZ_ERR_INVALID, "p: partition was not made for this context (rank/world/levels)");
  for (int l = 0; l < ctx->levels; ++l)
    if (p->group[l] != ctx->group[l]) return fail(HZ_ERR_INVALID, "p: group sizes differ from the context");
  if (!block_ok(p->block)) return fail(HZ_ERR_INVALID, "p.block: must be a power of two in [32, 2048]");
  if (p->padded_numel % (int64_t(p->world) * 4 * p->block))
    return fail(HZ_ERR_INVALID, "p.padded_numel: not a multiple of world*4*block");
  if (p->nhops < 0 || p->nhops > p->levels) return fail(HZ_ERR_INVALID, "p.nhops: must be in [0, levels]");
  for (int k = 0, prev = 0; k < p->nhops; prev = p->hop_last[k], ++k)
    if (p->hop_last[k] <= prev || p->hop_last[k] > p->levels || (k + 1 == p->nhops && p->hop_last[k] != p->levels))
      return fail(HZ_ERR_INVALID, "p.hop_last: must be strictly ascending and end at level L");
  return HZ_OK;
}

int64_t elem_bytes(hz_dtype dt) { return dt == HZ_F32 ? 4 : 2; }

namespace {
bool dtype_ok(hz_dtype dt) { return dt == HZ_F32 || dt == HZ_BF16 || dt == HZ_F16; }

ncclDataType_t nccl_dtype(hz_dtype dt) {
  return dt == HZ_F32 ? ncclFloat32 : (dt == HZ_BF16 ? ncclBfloat16 : ncclFloat16);
}

}  // namespace

// traced kernel launches ----------------------------------------------------
hz_status run_quantize(const void* x, hz_dtype dt, int64_t n, int bits, int block, uint8_t* c,
                       float* s, cudaStream_t st, int level, const SyncArgs* sync) {
  TraceScope t(st, "quantize", level, bits, n, n * elem_bytes(dt) + code_bytes(n, bits) + n / block * 4);
  SyncArgs sy = sync ? *sync : SyncArgs{};
  sy.stamps = t.stamps;
  cudaError_t e = launch_quantize(x, dt, n, bits, block, c, s, st, (sync || t.stamps) ? &sy : nullptr);
  t.end();
  if (e != cudaSuccess) return cuda_fail(e, "quantize kernel launch");
  return HZ_OK;
}

hz_status run_dequantize(const uint8_t* c, const float* s, int64_t n, int bits, int block, void* y,
                         hz_dtype odt, cudaStream_t st, int level) {
  TraceScope t(st, "dequantize", level, bits, n, code_bytes(n, bits) + n / block * 4 + n * elem_bytes(odt));
  Pieces pc{};
  pc.c[0] = c;
  pc.s[0] = s;
  pc.n = 1;
  pc.len = n;
  SyncArgs sy{};
  sy.stamps = t.stamps;
  cudaError_t e = launch_gather_dequantize(pc, n, bits, block, y, odt, st, t.stamps ? &sy : nullptr);
  t.end();
  if (e != cudaSuccess) return cuda_fail(e, "dequantize kernel launch");
  return HZ_OK;
}

hz_status run_gather_dequantize(const Pieces& pc, int64_t n, int bits, int block, void* y,
                                hz_dtype odt, cudaStream_t st, int level, const SyncArgs* sync,
                                int64_t remote_bytes) {
  TraceScope t(st, "gather_dequantize", level, bits, n,
               code_bytes(n, bits) + n / block * 4 + n * elem_bytes(odt) - remote_bytes, remote_bytes);
  SyncArgs sy = sync ? *sync : SyncArgs{};
  sy.stamps = t.stamps;
  cudaError_t e = launch_gather_dequantize(pc, n, bits, block, y, odt, st, (sync || t.stamps) ? &sy : nullptr);
  t.end();
  if (e != cudaSuccess) return cuda_fail(e, "gather-dequantize kernel launch");
  return HZ_OK;
}

hz_status run_gather_quantize(const Pieces& pc, int64_t n, int bits, void* y, hz_dtype odt, const void* x,
                              hz_dtype dt, int64_t nq, int qbits, uint8_t* c, float* s, cudaStream_t st,
                              const SyncArgs& sync, int64_t remote_bytes, float* qy, int acc) {
  const int64_t g_bytes = code_bytes(n, bits) + n / 256 * 4 + n * elem_bytes(odt) - remote_bytes;
  const int64_t q_bytes = nq * elem_bytes(dt) + (qy ? nq * 4 * (acc ? 2 : 1) : code_bytes(nq, qbits) + nq / 256 * 4);
  TraceScope t(st, qy ? "dequantize_roundtrip" : "gather_quantize", 0, bits, n + nq, g_bytes + q_bytes, remote_bytes);
  SyncArgs sy = sync;
  sy.stamps = t.stamps;
  cudaError_t e = launch_gather_quantize(pc, n, y, x, dt, nq, qbits, c, s, qy, acc, st, sy);
  t.end();
  if (e != cudaSuccess) return cuda_fail(e, "gather+quantize kernel launch");
  return HZ_OK;
}

hz_status run_gather_quantize_reduce(const Pieces& pc, int64_t n, void* y, const void* x, hz_dtype dt, int64_t nq,
                                     int qbits, uint8_t* c, float* s, int rg, const uint8_t* const* rc,
                                     const float* const* rs, int64_t rn, int rbits, float* shard, int acc, int level,
                                     cudaStream_t st, const SyncArgs& sync, int64_t remote_bytes) {
  const int64_t g_bytes = code_bytes(n, 8) + n / 256 * 4 + n * 2;
  const int64_t q_bytes = nq * elem_bytes(dt) + code_bytes(nq, qbits) + nq / 256 * 4;
  const int64_t r_bytes = rg * (code_bytes(rn, rbits) + rn / 256 * 4) + rn * 4 * (acc ? 2 : 1);
  TraceScope t(st, "gather_quantize_reduce", level, rbits, n + nq + rn, g_bytes + q_bytes + r_bytes - remote_bytes,
               remote_bytes);
  SyncArgs sy = sync;
  sy.stamps = t.stamps;
  cudaError_t e = launch_gather_quantize_reduce(pc, n, y, x, dt, nq, qbits, c, s, rg, rc, rs, rn, rbits, shard, acc,
                                                st, sy);
  t.end();
  if (e != cudaSuccess) return cuda_fail(e, "gather+quantize+reduce kernel launch");
  return HZ_OK;
}

hz_status run_reduce(int g, const uint8_t* const* c, const float* const* s, int64_t n, int bits_in,
                     int block, int bits_out, uint8_t* oc, float* os, float* of, int acc,
                     cudaStream_t st, int level, const SyncArgs* sync, int64_t remote_bytes) {
  const int64_t in_bytes = g * (code_bytes(n, bits_in) + n / block * 4);
  const int64_t out_bytes =
      bits_out ? code_bytes(n, bits_out) + n / block * 4 : n * 4 * (acc ? 2 : 1);
  TraceScope t(st, bits_out ? "reduce_requant" : "reduce", level, bits_in, n,
               in_bytes + out_bytes - remote_bytes, remote_bytes);
  SyncArgs sy = sync ? *sync : SyncArgs{};
  sy.stamps = t.stamps;
  cudaError_t e = launch_reduce(g, c, s, n, bits_in, block, bits_out, oc, os, of, acc, st,
                                (sync || t.stamps) ? &sy : nullptr);
  t.end();
  if (e != cudaSuccess) return cuda_fail(e, "reduce kernel launch");
  return HZ_OK;
}

hz_status run_roundtrip(const void* x, hz_dtype dt, int64_t n, int bits, int block, uint8_t* c, float* s,
                        void* y, hz_dtype odt, int acc, cudaStream_t st, int level) {
  const int64_t out = n * elem_bytes(odt) * (acc ? 2 : 1);
  TraceScope t(st, "quantize_dequantize", level, bits, n,
               n * elem_bytes(dt) + (c ? code_bytes(n, bits) + n / block * 4 : 0) + out);
  SyncArgs sy{};
  sy.stamps = t.stamps;
  cudaError_t e = launch_quantize_roundtrip(x, dt, n, bits, block, c, s, y, odt, acc, st, t.stamps ? &sy : nullptr);
  t.end();
  if (e != cudaSuccess) return cuda_fail(e, "quantize-dequantize kernel launch");
  return HZ_OK;
}

hz_status run_adamw(const float* g, float* th, float* m, float* v, void* out, hz_dtype dt, int64_t n,
                    const AdamW& hp, cudaStream_t st, const SyncArgs* sync) {
  TraceScope t(st, "adamw", 0, 32, n, n * (16 + 12 + elem_bytes(dt)));
  SyncArgs sy = sync ? *sync : SyncArgs{};
  sy.stamps = t.stamps;
  cudaError_t e = launch_adamw(g, th, m, v, out, dt, n, hp, st, (sync || t.stamps) ? &sy : nullptr);
  t.end();
  if (e != cudaSuccess) return cuda_fail(e, "adamw kernel launch");
  return HZ_OK;
}

hz_status run_sum(const Pieces& pc, int64_t n, float* out, cudaStream_t st, int level, const SyncArgs* sync,
                  int64_t remote) {
  TraceScope t(st, "allreduce_sum", level, 32, n, (pc.n + 1) * n * 4 - remote, remote);
  SyncArgs sy = sync ? *sync : SyncArgs{};
  sy.stamps = t.stamps;
  cudaError_t e = launch_sum_f32(pc, n, out, st, (sync || t.stamps) ? &sy : nullptr);
  t.end();
  if (e != cudaSuccess) return cuda_fail(e, "allreduce-sum kernel launch");
  return HZ_OK;
}

hz_status copy_async(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0 || dst == src) return HZ_OK;
  TraceScope t(st, "copy", 0, 0, 0, int64_t(bytes) * 2);
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st);
  t.end();
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync");
  return HZ_OK;
}

}  // namespace hz

extern "C" {

hz_status hz_get_uid(hz_uid* out) {
  using namespace hz;
  if (!out) return fail(HZ_ERR_INVALID, "out: NULL");
  static_assert(sizeof(ncclUniqueId) == sizeof(hz_uid), "hz_uid must be an ncclUniqueId");
  ncclUniqueId id;
  HZ_NCCL(ncclGetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out->bytes, &id, sizeof(id));
  clear_error();
  return HZ_OK;
}

hz_status hz_init(hz_ctx** out, int rank, int world, const hz_uid* uid, int levels,
                  const int* group, int cuda_device, size_t workspace_bytes) {
  using namespace hz;
  if (!out) return fail(HZ_ERR_INVALID, "out: NULL");
  *out = nullptr;
  if (!uid) return fail(HZ_ERR_INVALID, "uid: NULL");
  if (!group) return fail(HZ_ERR_INVALID, "group: NULL");
  if (levels < 1 || levels > HZ_MAX_LEVELS) return fail(HZ_ERR_INVALID, "levels: must be in [1, 4]");
  int64_t prod = 1;
  for (int l = 0; l < levels; ++l) {
    if (group[l] < 1) return fail(HZ_ERR_INVALID, "group[" + std::to_string(l) + "]: must be >= 1");
    prod *= group[l];
  }
  if (world < 1 || prod != world) return fail(HZ_ERR_INVALID, "group: product must equal world");
  if (rank < 0 || rank >= world) return fail(HZ_ERR_INVALID, "rank: must be in [0, world)");
  if (cuda_device < 0) return fail(HZ_ERR_INVALID, "cuda_device: negative");
  HZ_CUDA(cudaSetDevice(cuda_device), "cudaSetDevice");

  hz_ctx* ctx = new hz_ctx();
  ctx->rank = rank;
  ctx->world = world;
  ctx->levels = levels;
  ctx->device = cuda_device;
  ncclUniqueId id;
  std::memcpy(&id, uid->bytes, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&ctx->world_comm, world, id, rank);
  if (r != ncclSuccess) {
    delete ctx;
    return nccl_fail(r, "ncclCommInitRank");
  }
  int stride = 1;
  for (int l = 0; l < levels; ++l) {
    ctx->group[l] = group[l];
    ctx->digit[l] = (rank / stride) % group[l];
    if (group[l] > 1) {
      const int color = rank - ctx->digit[l] * stride;
      r = ncclCommSplit(ctx->world_comm, color, ctx->digit[l], &ctx->lvl[l], nullptr);
      if (r != ncclSuccess) {
        hz_finalize(ctx);
        return nccl_fail(r, "ncclCommSplit");
      }
    }
    stride *= group[l];
  }
  if (workspace_bytes) {
    hz_status st = grow(ctx->ag_c, workspace_bytes);
    if (st != HZ_OK) {
      hz_finalize(ctx);
      return st;
    }
  }
  *out = ctx;
  clear_error();
  return HZ_OK;
}

hz_status hz_finalize(hz_ctx* ctx) {
  using namespace hz;
  if (!ctx) return HZ_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  p2p_release(ctx);
  exec_release(ctx);
  for (int l = 0; l < HZ_MAX_LEVELS; ++l)
    if (ctx->lvl[l]) ncclCommDestroy(ctx->lvl[l]);
  for (auto& row : ctx->hop_comm)
    for (auto& c : row)
      if (c) ncclCommDestroy(c);
  if (ctx->world_comm) ncclCommDestroy(ctx->world_comm);
  for (auto* b : {&ctx->ag_c, &ctx->ag_s, &ctx->rs_a_c, &ctx->rs_a_s, &ctx->rs_b_c, &ctx->rs_b_s,
                  &ctx->rs_r_c, &ctx->rs_r_s, &ctx->ar_a, &ctx->ar_b, &ctx->ar_g})
    free_buf(*b);
  delete ctx;
  clear_error();
  return HZ_OK;
}

hz_status hz_partition(const hz_ctx* ctx, int64_t numel, int block, int w, int s, int gl,
                       hz_partition_t* out) {
  using namespace hz;
  if (!ctx) return fail(HZ_ERR_INVALID, "ctx: NULL");
  return partition(ctx->rank, ctx->levels, ctx->group, numel, block, w, s, gl, out);
}

static hz_status check_allgather(const hz_ctx* ctx, const hz_partition_t* p, int backward, const void* primary,
                                 hz_dtype dt, int bits, const uint8_t* sec_codes, const float* sec_scales,
                                 const void* full_out, hz_dtype out_dt) {
  using namespace hz;
  hz_status st0 = check_partition(ctx, p);
  if (st0 != HZ_OK) return st0;
  if (!bits_ok(bits)) return fail(HZ_ERR_INVALID, "bits: must be 4 or 8");
  if (!dtype_ok(out_dt)) return fail(HZ_ERR_INVALID, "out_dt: unknown dtype");
  if (!backward && !dtype_ok(dt)) return fail(HZ_ERR_INVALID, "dt: unknown dtype");
  if (!backward && (!primary || !aligned16(primary)))
    return fail(HZ_ERR_INVALID, "primary: NULL or not 16-byte aligned");
  if (!sec_codes || !aligned16(sec_codes)) return fail(HZ_ERR_INVALID, "sec_codes: NULL or not 16-byte aligned");
  if (!sec_scales || !aligned16(sec_scales)) return fail(HZ_ERR_INVALID, "sec_scales: NULL or not 16-byte aligned");
  if (!full_out || !aligned16(full_out)) return fail(HZ_ERR_INVALID, "full_out: NULL or not 16-byte aligned");
  return HZ_OK;
}

static hz_status allgather_impl(hz_ctx* ctx, const hz_partition_t* p, int backward, const void* primary,
                                hz_dtype dt, int bits, uint8_t* sec_codes, float* sec_scales, void* full_out,
                                hz_dtype out_dt, void* stream, const hz::NextQ* nextq);

hz_status hz_allgather_params(hz_ctx* ctx, const hz_partition_t* p, int backward,
                              const void* primary, hz_dtype dt, int bits, uint8_t* sec_codes,
                              float* sec_scales, void* full_out, hz_dtype out_dt, void* stream) {
  return allgather_impl(ctx, p, backward, primary, dt, bits, sec_codes, sec_scales, full_out, out_dt, stream,
                        nullptr);
}

hz_status hz_allgather_params_next(hz_ctx* ctx, const hz_partition_t* p, const void* primary, hz_dtype dt,
                                   int bits, uint8_t* sec_codes, float* sec_scales, void* full_out,
                                   hz_dtype out_dt, const hz_partition_t* p_next, const void* next_primary,
                                   uint8_t* next_sec_codes, float* next_sec_scales, void* stream) {
  using namespace hz;
  const CarveScope carve_scope(ctx ? ctx->world : 0);
  if (!p_next) return allgather_impl(ctx, p, 0, primary, dt, bits, sec_codes, sec_scales, full_out, out_dt, stream,
                                     nullptr);
  hz_status rc = check_partition(ctx, p_next);
  if (rc != HZ_OK) return fail(rc, std::string("p_next: ") + hz_last_error());
  if (p_next->block != p->block) return fail(HZ_ERR_INVALID, "p_next: block differs from p");
  if (!next_primary || !aligned16(next_primary))
    return fail(HZ_ERR_INVALID, "next_primary: NULL or not 16-byte aligned");
  if (!next_sec_codes || !aligned16(next_sec_codes))
    return fail(HZ_ERR_INVALID, "next_sec_codes: NULL or not 16-byte aligned");
  if (!next_sec_scales || !aligned16(next_sec_scales))
    return fail(HZ_ERR_INVALID, "next_sec_scales: NULL or not 16-byte aligned");
  NextQ nx{p_next, next_primary, next_sec_codes, next_sec_scales};
  return allgather_impl(ctx, p, 0, primary, dt, bits, sec_codes, sec_scales, full_out, out_dt, stream, &nx);
}

static hz_status allgather_impl(hz_ctx* ctx, const hz_partition_t* p, int backward, const void* primary,
                                hz_dtype dt, int bits, uint8_t* sec_codes, float* sec_scales, void* full_out,
                                hz_dtype out_dt, void* stream, const hz::NextQ* nextq) {
  using namespace hz;
  const CarveScope carve_scope(ctx ? ctx->world : 0);
  hz_status st0 = check_allgather(ctx, p, backward, primary, dt, bits, sec_codes, sec_scales, full_out, out_dt);
  if (st0 != HZ_OK) return st0;
  st0 = check_async(ctx);
  if (st0 != HZ_OK) return st0;

  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t Np = p->padded_numel;
  const int B = p->block;
  const int w = p->w, s = p->s;
  if (Np == 0) {
    clear_error();
    return HZ_OK;
  }
  if (ctx->p2p.on)   // NVLink peer-memory transport: fused gather + dequantize
    return p2p_allgather(ctx, p, backward, primary, dt, bits, sec_codes, sec_scales, full_out, out_dt, st, nextq);
  hz_status rc;
  if ((rc = grow(ctx->ag_c, code_bytes(Np, bits))) != HZ_OK) return rc;
  if ((rc = grow(ctx->ag_s, Np / B * 4)) != HZ_OK) return rc;
  uint8_t* ws_c = static_cast<uint8_t*>(ctx->ag_c.p);
  float* ws_s = static_cast<float*>(ctx->ag_s.p);

  const uint8_t* cur_c;
  const float* cur_s;
  int top;
  if (!backward && p->len[w] == Np && roundtrip_supported(B)) {
    // A2 + A5 fused: no level up to w exchanges anything (all its groups have one
    // member), so the gathered layer is the own quantized primary: one kernel writes
    // the codes (the secondary when it covers the same range) and the dequantized layer.
    const bool direct = p->len[s] == Np;
    uint8_t* qc = direct ? sec_codes : ws_c;
    float* qs = direct ? sec_scales : ws_s;
    if ((rc = run_roundtrip(primary, dt, Np, bits, B, qc, qs, full_out, out_dt, 0, st, w)) != HZ_OK) return rc;
    if (!direct) {   // A4, s > w: sub-slice of the quantized primary
      if ((rc = copy_async(sec_codes, qc + code_bytes(p->off[s], bits), code_bytes(p->len[s], bits), st)) != HZ_OK)
        return rc;
      if ((rc = copy_async(sec_scales, qs + p->off[s] / B, p->len[s] / B * 4, st)) != HZ_OK) return rc;
    }
    clear_error();
    return HZ_OK;
  }
  if (!backward) {
    // A2: quantize the primary range_w.  With s == w the quantized primary IS the
    // secondary (setting T, sec-degree = primary degree), so write it there.
    uint8_t* qc = s == w ? sec_codes : ws_c + code_bytes(p->off[w], bits);
    float* qs = s == w ? sec_scales : ws_s + p->off[w] / B;
    if ((rc = run_quantize(primary, dt, p->len[w], bits, B, qc, qs, st, w)) != HZ_OK) return rc;
    if (s > w) {   // A4, s > w: the secondary is a sub-slice of the own quantized primary
      const int64_t rel = p->off[s] - p->off[w];
      if ((rc = copy_async(sec_codes, qc + code_bytes(rel, bits), code_bytes(p->len[s], bits), st)) != HZ_OK) return rc;
      if ((rc = copy_async(sec_scales, qs + rel / B, p->len[s] / B * 4, st)) != HZ_OK) return rc;
    }
    cur_c = qc;
    cur_s = qs;
    top = w;
  } else {
    cur_c = sec_codes;   // O8: start from the secondary, no requantization
    cur_s = sec_scales;
    top = s;
  }
  std::vector<hz_comm_step> plan;
  if ((rc = plan_allgather(p, backward, bits, &plan)) != HZ_OK) return rc;
  size_t next = 0;
  for (int l = top; l >= 1; --l) {
    const int g = ctx->group[l - 1];
    if (next < plan.size() && plan[next].level == l) {   // A3: in-place all-gather of range_l pieces
      const hz_comm_step& step = plan[next++];             //     into range_{l-1}
      uint8_t* dc = ws_c + code_bytes(step.recv_off, bits);
      float* ds = ws_s + step.recv_off / B;
      const int64_t nb = step.code_bytes;
      const int64_t ns = step.scale_bytes / 4;
      TraceScope t(st, "nccl_allgather", l, bits, step.elems, (g - 1) * (nb + ns * 4));
      HZ_NCCL(ncclGroupStart(), "ncclGroupStart");
      HZ_NCCL(ncclAllGather(cur_c, dc, nb, ncclUint8, ctx->lvl[l - 1], st), "ncclAllGather(codes)");
      HZ_NCCL(ncclAllGather(cur_s, ds, ns, ncclFloat32, ctx->lvl[l - 1], st), "ncclAllGather(scales)");
      HZ_NCCL(ncclGroupEnd(), "ncclGroupEnd");
      t.end();
      cur_c = dc;
      cur_s = ds;
    }
    if (!backward && s < w && l - 1 == s) {   // A4, s < w: keep the intermediate range_s
      if ((rc = copy_async(sec_codes, cur_c, code_bytes(p->len[s], bits), st)) != HZ_OK) return rc;
      if ((rc = copy_async(sec_scales, cur_s, p->len[s] / B * 4, st)) != HZ_OK) return rc;
    }
  }
  // A5 / A6: every rank dequantizes the whole layer from the codes (R9).
  if ((rc = run_dequantize(cur_c, cur_s, Np, bits, B, full_out, out_dt, st, 0)) != HZ_OK) return rc;
  clear_error();
  return HZ_OK;
}

static hz_status check_reduce_scatter(const hz_ctx* ctx, const hz_partition_t* p, const void* grad, hz_dtype dt,
                                      int from_level, int to_level, const int* bits_per_level, const float* shard) {
  using namespace hz;
  hz_status rc = check_partition(ctx, p);
  if (rc != HZ_OK) return rc;
  const int L = ctx->levels;
  if (from_level < 1 || from_level > L) return fail(HZ_ERR_INVALID, "from_level: must be in [1, levels]");
  if (to_level < from_level || to_level > L) return fail(HZ_ERR_INVALID, "to_level: must be in [from_level, levels]");
  if (!bits_per_level) return fail(HZ_ERR_INVALID, "bits_per_level: NULL");
  for (int l = from_level; l <= to_level; ++l)
    if (!bits_ok(bits_per_level[l - 1]))
      return fail(HZ_ERR_INVALID, "bits_per_level[" + std::to_string(l - 1) + "]: must be 4 or 8");
  if (!dtype_ok(dt)) return fail(HZ_ERR_INVALID, "dt: unknown dtype");
  if (!grad || !aligned16(grad)) return fail(HZ_ERR_INVALID, "grad: NULL or not 16-byte aligned");
  if (!shard || !aligned16(shard)) return fail(HZ_ERR_INVALID, "shard: NULL or not 16-byte aligned");
  std::vector<Hop> hops;
  return hops_of(p, from_level, to_level, &hops);
}

hz_status hz_backward_step(hz_ctx* ctx, const hz_partition_t* p, const void* grad, hz_dtype dt, int from_level,
                           int to_level, const int* bits_per_level, float* shard, int accumulate,
                           const hz_partition_t* p_prev, uint8_t* prev_sec_codes, float* prev_sec_scales,
                           int prev_bits, void* prev_full_out, hz_dtype prev_out_dt, void* stream) {
  using namespace hz;
  const CarveScope carve_scope(ctx ? ctx->world : 0);
  hz_status rc = check_reduce_scatter(ctx, p, grad, dt, from_level, to_level, bits_per_level, shard);
  if (rc != HZ_OK) return rc;
  if (!p_prev)
    return hz_reduce_scatter_grads(ctx, p, grad, dt, from_level, to_level, bits_per_level, shard, accumulate, stream);
  if ((rc = check_allgather(ctx, p_prev, 1, nullptr, HZ_BF16, prev_bits, prev_sec_codes, prev_sec_scales,
                            prev_full_out, prev_out_dt)) != HZ_OK)
    return fail(rc, std::string("prev: ") + hz_last_error());
  if ((rc = check_async(ctx)) != HZ_OK) return rc;
  PrevG pg{p_prev, prev_sec_codes, prev_sec_scales, prev_bits, prev_full_out, prev_out_dt};
  if (prev_full_out == grad) return fail(HZ_ERR_INVALID, "prev_full_out: aliases grad");
  if (ctx->p2p.on && p->len[from_level - 1] > 0 && p_prev->padded_numel > 0 &&
      p2p_prev_fusable(ctx, p, from_level, pg))
    return p2p_reduce_scatter(ctx, p, grad, dt, from_level, to_level, bits_per_level, shard, accumulate,
                              static_cast<cudaStream_t>(stream), &pg);
  if (!ctx->p2p.on && from_level == to_level && ctx->group[from_level - 1] == 1 && roundtrip_supported(p->block) &&
      p_prev->block == 256 && p_prev->len[p_prev->s] == p_prev->padded_numel && p_prev->padded_numel > 0 &&
      p->len[from_level - 1] > 0 && gather_quantize_supported(256, prev_bits, prev_out_dt) &&
      tune_param("pair1", 0) == 1) {
    // no exchange on either side (one-member groups): the previous layer's backward
    // gather is the dequantize of its secondary and this layer's qgZ the round trip of
    // its gradient — both HBM streams, one launch instead of two.  Off by default
    // (HZ_TUNE pair1=1): measured at N = 1, GPT-1.3B, 3.295 vs 3.270 ms per step — two
    // HBM-bound streams gain nothing from sharing a launch (profiles/pairing_r01/)
    Pieces pc{};
    pc.n = 1;
    pc.len = p_prev->padded_numel;
    pc.c[0] = prev_sec_codes;
    pc.s[0] = prev_sec_scales;
    if ((rc = run_gather_quantize(pc, p_prev->padded_numel, prev_bits, prev_full_out, prev_out_dt, grad, dt,
                                  p->len[from_level - 1], bits_per_level[from_level - 1], nullptr, nullptr,
                                  static_cast<cudaStream_t>(stream), SyncArgs{}, 0, shard, accumulate)) != HZ_OK)
      return rc;
    clear_error();
    return HZ_OK;
  }
  // not fusable (NCCL transport, other block sizes / dtypes): the two calls in order
  if ((rc = hz_allgather_params(ctx, p_prev, 1, nullptr, HZ_BF16, prev_bits, prev_sec_codes, prev_sec_scales,
                                prev_full_out, prev_out_dt, stream)) != HZ_OK)
    return rc;
  return hz_reduce_scatter_grads(ctx, p, grad, dt, from_level, to_level, bits_per_level, shard, accumulate, stream);
}

hz_status hz_reduce_scatter_grads(hz_ctx* ctx, const hz_partition_t* p, const void* grad,
                                  hz_dtype dt, int from_level, int to_level,
                                  const int* bits_per_level, float* shard, int accumulate,
                                  void* stream) {
  using namespace hz;
  const CarveScope carve_scope(ctx ? ctx->world : 0);
  hz_status rc = check_reduce_scatter(ctx, p, grad, dt, from_level, to_level, bits_per_level, shard);
  if (rc != HZ_OK) return rc;
  if ((rc = check_async(ctx)) != HZ_OK) return rc;

  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int B = p->block;
  const int64_t base_len = p->len[from_level - 1];
  if (base_len == 0) {
    clear_error();
    return HZ_OK;
  }
  if (ctx->p2p.on)   // NVLink peer-memory transport: reduce reads the peers' chunks in place
    return p2p_reduce_scatter(ctx, p, grad, dt, from_level, to_level, bits_per_level, shard, accumulate, st);
  if ((rc = grow(ctx->rs_a_c, base_len)) != HZ_OK) return rc;
  if ((rc = grow(ctx->rs_a_s, base_len / B * 4)) != HZ_OK) return rc;
  if ((rc = grow(ctx->rs_b_c, base_len)) != HZ_OK) return rc;
  if ((rc = grow(ctx->rs_b_s, base_len / B * 4)) != HZ_OK) return rc;
  if ((rc = grow(ctx->rs_r_c, base_len)) != HZ_OK) return rc;
  if ((rc = grow(ctx->rs_r_s, base_len / B * 4)) != HZ_OK) return rc;
  uint8_t* a_c = static_cast<uint8_t*>(ctx->rs_a_c.p);
  float* a_s = static_cast<float*>(ctx->rs_a_s.p);
  uint8_t* b_c = static_cast<uint8_t*>(ctx->rs_b_c.p);
  float* b_s = static_cast<float*>(ctx->rs_b_s.p);
  uint8_t* r_c = static_cast<uint8_t*>(ctx->rs_r_c.p);
  float* r_s = static_cast<float*>(ctx->rs_r_s.p);

  std::vector<Hop> hops;
  if ((rc = hops_of(p, from_level, to_level, &hops)) != HZ_OK) return rc;
  std::vector<int> ranks;
  std::vector<int64_t> rel;
  int me = 0;
  hop_members(p, hops[0].a, hops[0].b, &ranks, &rel, &me);
  if (hops.size() == 1 && ranks.size() == 1 && roundtrip_supported(B)) {
    // A7 + A9 fused: a single hop whose group has one member exchanges nothing, so
    // the shard is the round trip of the own gradient: one kernel, codes never reread.
    // (the gradient's codes are never read by anyone here, so they are not stored)
    if ((rc = run_roundtrip(grad, dt, base_len, bits_per_level[from_level - 1], B, nullptr, nullptr, shard, HZ_F32,
                            accumulate, st, from_level)) != HZ_OK)
      return rc;
    clear_error();
    return HZ_OK;
  }
  // A7: quantize the whole input range_{from-1}; the chunk of member j goes to j.
  if ((rc = run_quantize(grad, dt, base_len, bits_per_level[from_level - 1], B, a_c, a_s, st,
                         from_level)) != HZ_OK)
    return rc;
  std::vector<hz_comm_step> plan;
  if ((rc = plan_reduce_scatter(p, from_level, to_level, bits_per_level, &plan)) != HZ_OK) return rc;
  size_t next = 0;
  for (size_t h = 0; h < hops.size(); ++h) {
    const Hop& hp = hops[h];
    hop_members(p, hp.a, hp.b, &ranks, &rel, &me);
    const int g = static_cast<int>(ranks.size());
    const int bits = bits_per_level[hp.a - 1];
    const int64_t cl = p->len[hp.b];
    const int64_t cb = code_bytes(cl, bits);
    const int64_t cs = cl / B;
    if (g > kMaxG) return fail(HZ_ERR_UNSUPPORTED, "more than 16 ranks in one qgZ hop");
    const uint8_t* ptr_c[kMaxG];
    const float* ptr_s[kMaxG];
    if (g > 1) {   // A8: all-to-all within the hop group, from the plan
      ncclComm_t comm = nullptr;
      if ((rc = hop_comm(ctx, hp.a, hp.b, &comm)) != HZ_OK) return rc;
      TraceScope t(st, "nccl_alltoall", hp.b, bits, cl, (g - 1) * (cb + cs * 4));
      HZ_NCCL(ncclGroupStart(), "ncclGroupStart");
      for (; next < plan.size() && plan[next].level == hp.a; ++next) {
        const hz_comm_step& s = plan[next];
        const int j = s.peer;
        const int64_t relj = s.send_off - p->off[hp.a - 1];   // member j's chunk of this rank's range_{a-1}
        HZ_NCCL(ncclSend(a_c + code_bytes(relj, bits), s.code_bytes, ncclUint8, j, comm, st), "ncclSend(codes)");
        HZ_NCCL(ncclRecv(r_c + j * cb, s.code_bytes, ncclUint8, j, comm, st), "ncclRecv(codes)");
        HZ_NCCL(ncclSend(a_s + relj / B, s.scale_bytes / 4, ncclFloat32, j, comm, st), "ncclSend(scales)");
        HZ_NCCL(ncclRecv(r_s + j * cs, s.scale_bytes / 4, ncclFloat32, j, comm, st), "ncclRecv(scales)");
      }
      HZ_NCCL(ncclGroupEnd(), "ncclGroupEnd");
      t.end();
    }
    for (int j = 0; j < g; ++j) {
      ptr_c[j] = j == me ? a_c + code_bytes(rel[me], bits) : r_c + j * cb;
      ptr_s[j] = j == me ? a_s + rel[me] / B : r_s + j * cs;
    }
    if (h + 1 < hops.size()) {   // A9 fused with the next hop's requantization
      if ((rc = run_reduce(g, ptr_c, ptr_s, cl, bits, B, bits_per_level[hops[h + 1].a - 1], b_c, b_s, nullptr, 0, st,
                           hp.b)) != HZ_OK)
        return rc;
      std::swap(a_c, b_c);
      std::swap(a_s, b_s);
    } else {                     // A9/A10: final fp32 shard, optionally accumulated
      if ((rc = run_reduce(g, ptr_c, ptr_s, cl, bits, B, 0, nullptr, nullptr, shard, accumulate, st, hp.b)) != HZ_OK)
        return rc;
    }
  }
  clear_error();
  return HZ_OK;
}

hz_status hz_allreduce_select(hz_ctx* ctx, const hz_partition_t* p, const float* shard_in, int from_level,
                              int to_level, float* out, void* stream) {
  using namespace hz;
  hz_status rc = check_partition(ctx, p);
  if (rc != HZ_OK) return rc;
  const int L = ctx->levels;
  if (from_level < 1 || from_level > L) return fail(HZ_ERR_INVALID, "from_level: must be in [1, levels]");
  if (to_level < from_level || to_level > L) return fail(HZ_ERR_INVALID, "to_level: must be in [from_level, levels]");
  if (!shard_in || !aligned16(shard_in)) return fail(HZ_ERR_INVALID, "shard_in: NULL or not 16-byte aligned");
  if (!out || !aligned16(out)) return fail(HZ_ERR_INVALID, "out: NULL or not 16-byte aligned");
  if ((rc = check_async(ctx)) != HZ_OK) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = p->len[from_level - 1];
  const int64_t sel = p->off[to_level] - p->off[from_level - 1];
  if (n == 0) {
    clear_error();
    return HZ_OK;
  }
  if (ctx->p2p.on) return p2p_allreduce_select(ctx, p, shard_in, from_level, to_level, out, st);
  // NCCL transport: per level, all-gather the members' full buffers (piece j = digit
  // j) and sum them locally in ascending digit — the oracle's order, bit for bit
  const size_t nb = static_cast<size_t>(n) * 4;
  if ((rc = grow(ctx->ar_a, nb)) != HZ_OK) return rc;
  if ((rc = grow(ctx->ar_b, nb)) != HZ_OK) return rc;
  int gmax = 1;
  for (int l = from_level; l <= to_level; ++l) gmax = ctx->group[l - 1] > gmax ? ctx->group[l - 1] : gmax;
  if ((rc = grow(ctx->ar_g, nb * gmax)) != HZ_OK) return rc;
  const float* cur = shard_in;
  float* bufs[2] = {static_cast<float*>(ctx->ar_a.p), static_cast<float*>(ctx->ar_b.p)};
  int nxt = 0;
  for (int l = from_level; l <= to_level; ++l) {
    const int g = ctx->group[l - 1];
    if (g == 1) continue;
    float* G = static_cast<float*>(ctx->ar_g.p);
    {
      TraceScope t(st, "nccl_allgather", l, 32, n * g, nb * g, nb * (g - 1));
      ncclResult_t r = ncclAllGather(cur, G, n, ncclFloat32, ctx->lvl[l - 1], st);
      t.end();
      if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather(allreduce)");
    }
    Pieces pc{};
    pc.n = g;
    pc.len = n;
    for (int j = 0; j < g; ++j) pc.c[j] = reinterpret_cast<const uint8_t*>(G + j * n);
    if ((rc = run_sum(pc, n, bufs[nxt], st, l, nullptr, 0)) != HZ_OK) return rc;
    cur = bufs[nxt];
    nxt ^= 1;
  }
  if ((rc = copy_async(out, cur + sel, static_cast<size_t>(p->len[to_level]) * 4, st)) != HZ_OK) return rc;
  clear_error();
  return HZ_OK;
}

hz_status hz_adamw_params(double lr, double b1, double b2, double eps, double weight_decay, int64_t t,
                          hz_adamw_t* out) {
  using namespace hz;
  if (!out) return fail(HZ_ERR_INVALID, "out: NULL");
  if (t < 1) return fail(HZ_ERR_INVALID, "t: must be >= 1");
  if (!(b1 >= 0.0 && b1 < 1.0)) return fail(HZ_ERR_INVALID, "b1: must be in [0, 1)");
  if (!(b2 >= 0.0 && b2 < 1.0)) return fail(HZ_ERR_INVALID, "b2: must be in [0, 1)");
  // reading R19: every constant computed in double, rounded once to fp32
  const double td = static_cast<double>(t);
  out->b1 = static_cast<float>(b1);
  out->omb1 = static_cast<float>(1.0 - b1);
  out->b2 = static_cast<float>(b2);
  out->omb2 = static_cast<float>(1.0 - b2);
  out->lr_wd = static_cast<float>(lr * weight_decay);
  out->sqrt_bc2 = static_cast<float>(std::sqrt(1.0 - std::pow(b2, td)));
  out->eps = static_cast<float>(eps);
  out->step = static_cast<float>(lr / (1.0 - std::pow(b1, td)));
  clear_error();
  return HZ_OK;
}

hz_status hz_adamw_step(hz_ctx* ctx, const hz_partition_t* p, const float* grad_shard, float* master,
                        float* m, float* v, const hz_adamw_t* hp, void* primary, hz_dtype dt, void* stream) {
  using namespace hz;
  hz_status rc = check_partition(ctx, p);
  if (rc != HZ_OK) return rc;
  if (!hp) return fail(HZ_ERR_INVALID, "hp: NULL");
  if (!dtype_ok(dt)) return fail(HZ_ERR_INVALID, "dt: unknown dtype");
  for (const void* q : {static_cast<const void*>(grad_shard), static_cast<const void*>(master),
                        static_cast<const void*>(m), static_cast<const void*>(v), static_cast<const void*>(primary)})
    if (!q || !aligned16(q)) return fail(HZ_ERR_INVALID, "grad_shard/master/m/v/primary: NULL or not 16-byte aligned");
  if ((rc = check_async(ctx)) != HZ_OK) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int L = p->levels, w = p->w;
  const int64_t lenL = p->len[L];
  if (lenL == 0) {
    clear_error();
    return HZ_OK;
  }
  AdamW a{hp->b1, hp->omb1, hp->b2, hp->omb2, hp->lr_wd, hp->sqrt_bc2, hp->eps, hp->step};
  if (ctx->p2p.on) return p2p_adamw_gather(ctx, p, grad_shard, master, m, v, a, primary, dt, st);
  // the update lands in its place inside the primary; levels L..w+1 then gather in place
  char* prim = static_cast<char*>(primary);
  const int64_t eb = elem_bytes(dt);
  if ((rc = run_adamw(grad_shard, master, m, v, prim + (p->off[L] - p->off[w]) * eb, dt, lenL, a, st, nullptr)) !=
      HZ_OK)
    return rc;
  for (int l = L; l > w; --l) {
    const int g = ctx->group[l - 1];
    if (g <= 1) continue;
    TraceScope t(st, "nccl_allgather", l, 16, p->len[l], (g - 1) * p->len[l] * eb);
    HZ_NCCL(ncclAllGather(prim + (p->off[l] - p->off[w]) * eb, prim + (p->off[l - 1] - p->off[w]) * eb,
                          p->len[l], nccl_dtype(dt), ctx->lvl[l - 1], st),
            "ncclAllGather(updated weights)");
    t.end();
  }
  clear_error();
  return HZ_OK;
}

hz_status hz_flat_allgather(hz_ctx* ctx, const void* chunk, void* out, int64_t numel, hz_dtype dt,
                            void* stream) {
  using namespace hz;
  if (!ctx) return fail(HZ_ERR_INVALID, "ctx: NULL");
  if (!dtype_ok(dt)) return fail(HZ_ERR_INVALID, "dt: unknown dtype");
  if (numel < 0 || numel % ctx->world) return fail(HZ_ERR_INVALID, "numel: must be a non-negative multiple of world");
  if (!chunk || !out) return fail(HZ_ERR_INVALID, "chunk/out: NULL");
  hz_status rc = check_async(ctx);
  if (rc != HZ_OK) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t c = numel / ctx->world;
  TraceScope t(st, "nccl_flat", 0, 16, numel, (ctx->world - 1) * c * elem_bytes(dt));
  HZ_NCCL(ncclAllGather(chunk, out, c, nccl_dtype(dt), ctx->world_comm, st), "ncclAllGather");
  t.end();
  clear_error();
  return HZ_OK;
}

hz_status hz_flat_reduce_scatter(hz_ctx* ctx, const void* in, void* out_chunk, int64_t numel,
                                 hz_dtype dt, void* stream) {
  using namespace hz;
  if (!ctx) return fail(HZ_ERR_INVALID, "ctx: NULL");
  if (!dtype_ok(dt)) return fail(HZ_ERR_INVALID, "dt: unknown dtype");
  if (numel < 0 || numel % ctx->world) return fail(HZ_ERR_INVALID, "numel: must be a non-negative multiple of world");
  if (!in || !out_chunk) return fail(HZ_ERR_INVALID, "in/out_chunk: NULL");
  hz_status rc = check_async(ctx);
  if (rc != HZ_OK) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t c = numel / ctx->world;
  TraceScope t(st, "nccl_flat", 0, 16, numel, (ctx->world - 1) * c * elem_bytes(dt));
  HZ_NCCL(ncclReduceScatter(in, out_chunk, c, nccl_dtype(dt), ncclSum, ctx->world_comm, st),
          "ncclReduceScatter");
  t.end();
  clear_error();
  return HZ_OK;
}

}  // extern "C"
