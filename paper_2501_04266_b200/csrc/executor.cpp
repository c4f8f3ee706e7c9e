// Host-staged step executor (hz_step_host): one step of the hot path whose inputs
// and results live in host memory.  Per-layer phase order of the paper's step
// (gather before forward, gather from the secondary before backward,
// reduce-scatter the gradients), one micro-batch.
//
// Three streams: host->device copies (library-owned), kernels (the caller's
// stream), device->host copies (library-owned).  Events per tensor:
//   ev[3i]   primary i uploaded      (h2d -> kernels)
//   ev[3i+1] gradient i uploaded     (h2d -> kernels)
//   ev[3i+2] shard i reduced         (kernels -> d2h)
// The uploads are issued in consumption order (primaries 0..n-1, then gradients
// n-1..0), so the kernels of tensor i start as soon as its bytes are on the GPU
// and the download of shard i overlaps the upload of gradient i-1.  A call's
// uploads wait only for the previous call's kernels (its staging buffers were
// read by them), not for its downloads: back-to-back steps keep both PCIe directions
// busy.  The kernel stream waits for the last download at the end, so
// the call is stream-ordered on `stream` like every other entry point.  Every argument
// (partitions, alignment, P2P-pool secondaries) is validated before anything is
// enqueued.  The kernels
// are issued as the paired calls (hz_allgather_params_next / hz_backward_step).
#include <string>

#include "ctx.h"

namespace hz {
namespace {

hz_status bad(int i, const char* field, const char* why) {
  return fail(HZ_ERR_INVALID, "t[" + std::to_string(i) + "]." + field + ": " + why);
}

hz_status ensure_exec(hz_ctx* ctx, int n) {
  auto& ex = ctx->exec;
  cudaError_t e = cudaSuccess;
  if (!ex.h2d) {
    if ((e = cudaStreamCreateWithFlags(&ex.h2d, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&ex.d2h, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ex.kernels_done, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ex.d2h_done, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_fail(e, "hz_step_host: stream / event creation");
  }
  while (ex.ev.size() < size_t(3) * n) {
    cudaEvent_t ev;
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_fail(e, "hz_step_host: cudaEventCreate");
    ex.ev.push_back(ev);
  }
  return HZ_OK;
}

}  // namespace

void exec_release(hz_ctx* ctx) {
  auto& ex = ctx->exec;
  for (cudaEvent_t e : ex.ev) cudaEventDestroy(e);
  ex.ev.clear();
  if (ex.kernels_done) cudaEventDestroy(ex.kernels_done);
  if (ex.d2h_done) cudaEventDestroy(ex.d2h_done);
  if (ex.h2d) cudaStreamDestroy(ex.h2d);
  if (ex.d2h) cudaStreamDestroy(ex.d2h);
  ex = hz_ctx::Exec{};
}

}  // namespace hz

extern "C" hz_status hz_step_host(hz_ctx* ctx, int n, const hz_tensor_io* t, hz_dtype dt, int qwz_bits,
                                  const int* qgz_bits, void* full_out0, void* full_out1, hz_dtype out_dt,
                                  void* stream) {
  using namespace hz;
  if (!ctx) return fail(HZ_ERR_INVALID, "ctx: NULL");
  if (n < 1) return fail(HZ_ERR_INVALID, "n: must be >= 1");
  if (!t) return fail(HZ_ERR_INVALID, "t: NULL");
  if (!bits_ok(qwz_bits)) return fail(HZ_ERR_INVALID, "qwz_bits: must be 4 or 8");
  if (!qgz_bits) return fail(HZ_ERR_INVALID, "qgz_bits: NULL");
  for (int l = 0; l < ctx->levels; ++l)
    if (!bits_ok(qgz_bits[l])) return fail(HZ_ERR_INVALID, "qgz_bits[" + std::to_string(l) + "]: must be 4 or 8");
  if (dt != HZ_F32 && dt != HZ_BF16 && dt != HZ_F16) return fail(HZ_ERR_INVALID, "dt: unknown dtype");
  if (out_dt != HZ_F32 && out_dt != HZ_BF16 && out_dt != HZ_F16)
    return fail(HZ_ERR_INVALID, "out_dt: unknown dtype");
  if (!full_out0 || !aligned16(full_out0)) return fail(HZ_ERR_INVALID, "full_out0: NULL or not 16-byte aligned");
  if (!full_out1 || !aligned16(full_out1)) return fail(HZ_ERR_INVALID, "full_out1: NULL or not 16-byte aligned");
  for (int i = 0; i < n; ++i) {
    const hz_tensor_io& x = t[i];
    const hz_partition_t* p = x.p;
    if (!p) return bad(i, "p", "NULL");
    if (check_partition(ctx, p) != HZ_OK) return bad(i, "p", hz_last_error());
    if (!x.h_primary) return bad(i, "h_primary", "NULL");
    if (!x.h_grad) return bad(i, "h_grad", "NULL");
    if (!x.h_shard) return bad(i, "h_shard", "NULL");
    if (!x.d_primary || !aligned16(x.d_primary)) return bad(i, "d_primary", "NULL or not 16-byte aligned");
    if (!x.d_grad || !aligned16(x.d_grad)) return bad(i, "d_grad", "NULL or not 16-byte aligned");
    if (!x.d_shard || !aligned16(x.d_shard)) return bad(i, "d_shard", "NULL or not 16-byte aligned");
    if (!x.sec_codes || !aligned16(x.sec_codes)) return bad(i, "sec_codes", "NULL or not 16-byte aligned");
    if (!x.sec_scales || !aligned16(x.sec_scales)) return bad(i, "sec_scales", "NULL or not 16-byte aligned");
    if (ctx->p2p.on) {   // peers read the secondaries in place: symmetric-pool memory (hz_sym_alloc)
      const int64_t ls = p->len[p->s];
      if (!in_pool(ctx, x.sec_codes, size_t(ls) * qwz_bits / 8))
        return bad(i, "sec_codes", "not hz_sym_alloc memory of the P2P pool (or too small)");
      if (!in_pool(ctx, x.sec_scales, size_t(ls / p->block) * 4))
        return bad(i, "sec_scales", "not hz_sym_alloc memory of the P2P pool (or too small)");
    }
  }
  hz_status rc = ensure_exec(ctx, n);
  if (rc != HZ_OK) return rc;

  auto& ex = ctx->exec;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t eb = elem_bytes(dt);
  const int L = ctx->levels;
  cudaError_t e = cudaSuccess;
#define HZ_X(call, what)                                  \
  do {                                                    \
    if ((e = (call)) != cudaSuccess) return cuda_fail(e, what); \
  } while (0)

  // uploads: after the previous call's kernels (not its downloads: back-to-back calls keep
  // both PCIe directions busy), in consumption order.  The staging buffers d_primary /
  // d_grad belong to the executor between calls (hz.h).  Measured: waiting instead for
  // everything on `stream` (an entry event, which includes the previous call's downloads)
  // cost 24 ms of 134 ms per GPT-1.3B step at N = 1.
  HZ_X(cudaStreamWaitEvent(ex.h2d, ex.kernels_done, 0), "hz_step_host: wait previous kernels");
  for (int i = 0; i < n; ++i) {
    const hz_partition_t* p = t[i].p;
    HZ_X(cudaMemcpyAsync(t[i].d_primary, t[i].h_primary, size_t(p->len[p->w] * eb), cudaMemcpyHostToDevice,
                         ex.h2d), "hz_step_host: primary upload");
    HZ_X(cudaEventRecord(ex.ev[3 * i], ex.h2d), "hz_step_host: cudaEventRecord");
  }
  for (int i = n - 1; i >= 0; --i) {
    const hz_partition_t* p = t[i].p;
    HZ_X(cudaMemcpyAsync(t[i].d_grad, t[i].h_grad, size_t(p->padded_numel * eb), cudaMemcpyHostToDevice,
                         ex.h2d), "hz_step_host: gradient upload");
    HZ_X(cudaEventRecord(ex.ev[3 * i + 1], ex.h2d), "hz_step_host: cudaEventRecord");
  }

  void* full[2] = {full_out0, full_out1};
  // forward: gather layer i with the quantize of layer i+1 prefetched into the same
  // launch (hz_allgather_params_next), as soon as both primaries are on the GPU
  HZ_X(cudaStreamWaitEvent(st, ex.ev[0], 0), "hz_step_host: wait primary");
  for (int i = 0; i < n; ++i) {
    const bool nx = i + 1 < n;
    if (nx) HZ_X(cudaStreamWaitEvent(st, ex.ev[3 * (i + 1)], 0), "hz_step_host: wait primary");
    rc = hz_allgather_params_next(ctx, t[i].p, t[i].d_primary, dt, qwz_bits, t[i].sec_codes, t[i].sec_scales,
                                  full[i & 1], out_dt, nx ? t[i + 1].p : nullptr, nx ? t[i + 1].d_primary : nullptr,
                                  nx ? t[i + 1].sec_codes : nullptr, nx ? t[i + 1].sec_scales : nullptr, stream);
    if (rc != HZ_OK) return rc;
  }
  // backward: layer i's qgZ with layer i-1's gather from its secondary (hz_backward_step),
  // then the download of layer i's shard
  rc = hz_allgather_params(ctx, t[n - 1].p, 1, nullptr, dt, qwz_bits, t[n - 1].sec_codes, t[n - 1].sec_scales,
                           full[(n - 1) & 1], out_dt, stream);
  if (rc != HZ_OK) return rc;
  for (int i = n - 1; i >= 0; --i) {
    const hz_partition_t* p = t[i].p;
    HZ_X(cudaStreamWaitEvent(st, ex.ev[3 * i + 1], 0), "hz_step_host: wait gradient");
    const bool pv = i > 0;
    rc = hz_backward_step(ctx, p, t[i].d_grad, dt, 1, L, qgz_bits, t[i].d_shard, 0, pv ? t[i - 1].p : nullptr,
                          pv ? t[i - 1].sec_codes : nullptr, pv ? t[i - 1].sec_scales : nullptr, qwz_bits,
                          pv ? full[(i - 1) & 1] : nullptr, out_dt, stream);
    if (rc != HZ_OK) return rc;
    // P2P transport: hz_backward_step with a previous layer defers its last qgZ hop into
    // the next call's launch, so layer i+1's shard is complete once this call is enqueued
    // (and, after the last call, layer 0's as well)
    int ready[2], nready = 0;
    if (i + 1 <= n - 1) ready[nready++] = i + 1;
    if (i == 0) ready[nready++] = 0;
    for (int k = 0; k < nready; ++k) {
      const int j = ready[k];
      HZ_X(cudaEventRecord(ex.ev[3 * j + 2], st), "hz_step_host: cudaEventRecord");
      HZ_X(cudaStreamWaitEvent(ex.d2h, ex.ev[3 * j + 2], 0), "hz_step_host: wait shard");
      HZ_X(cudaMemcpyAsync(t[j].h_shard, t[j].d_shard, size_t(t[j].p->len[L] * 4), cudaMemcpyDeviceToHost,
                           ex.d2h),
           "hz_step_host: shard download");
    }
  }
  HZ_X(cudaEventRecord(ex.kernels_done, st), "hz_step_host: cudaEventRecord");
  HZ_X(cudaEventRecord(ex.d2h_done, ex.d2h), "hz_step_host: cudaEventRecord");
  HZ_X(cudaStreamWaitEvent(st, ex.d2h_done, 0), "hz_step_host: wait downloads");
#undef HZ_X
  clear_error();
  return HZ_OK;
}
