// Virtual world (hz_init_virtual): W hz contexts in ONE process on ONE GPU (or, with
// hz_init_virtual_ex, on several GPUs of this process with peer access), whose
// "peer" pools are each other's allocations — the product's P2P exchange kernels,
// flags and phase protocol, without IPC or NCCL.  It exists so that the multi-rank
// path (multi-piece gathers, hop groups, the level-local protocol) can be checked
// bit for bit against the oracle on a single GPU.
//
// The W contexts are driven by W host threads, one stream each.  On one GPU their
// spin-waiting kernels could deadlock: a kernel whose producer sits behind it in a
// shared hardware queue, or waits for SMs the waiter occupies, never starts.  So
// every synchronised launch is also ordered on the host: before launching a kernel
// that waits for ready/done phases from ranks q, the calling thread blocks until
// those ranks have enqueued the kernels that signal them and makes its stream wait
// on their CUDA events; after launching a kernel that signals, it records an event.
// Every kernel therefore starts only after its producers completed, its device-side
// wait passes at once (the flags it checks are the real ones), and there is no
// co-residency requirement.  A host wait longer than the context's timeout aborts the
// context (HZ_ERR_ABORTED), like a device-side timeout.
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>

#include "ctx.h"

namespace hz {

struct VWorld {
  struct Ev {
    cudaEvent_t e = nullptr;
    ~Ev() {
      if (e) cudaEventDestroy(e);
    }
  };
  struct Ent {
    unsigned long long v;
    std::shared_ptr<Ev> ev;
  };
  int world = 0;
  int refs = 0;
  std::mutex mu;
  std::condition_variable cv;
  bool aborted = false;
  std::deque<Ent> ready[kMaxWorld][kMaxWorld];   // [source][target]
  std::deque<Ent> done[kMaxWorld][kMaxWorld];
  char* pools[kMaxWorld] = {nullptr};
  int devices[kMaxWorld] = {0};
};

namespace {

// the first entry of q's signals to `me` with value >= v; older entries are dropped
// (thresholds of one target are nondecreasing)
const VWorld::Ent* find(std::deque<VWorld::Ent>& dq, unsigned long long v) {
  while (!dq.empty() && dq.front().v < v) {
    if (dq.size() == 1) return nullptr;   // keep the latest (a later wait may need no newer one)
    dq.pop_front();
  }
  return dq.empty() ? nullptr : &dq.front();
}

}  // namespace

hz_status vw_wait(hz_ctx* ctx, const SyncArgs& s, cudaStream_t st) {
  VWorld* vw = ctx->p2p.vw;
  const unsigned long long e = ctx->p2p.epoch_host;   // 0: no graphs in a virtual world
  const unsigned long long wr = s.wait_ready + e, wd = s.wait_done + e;
  const int me = ctx->rank;
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::nanoseconds(ctx->p2p.timeout_ns);
  std::unique_lock<std::mutex> lock(vw->mu);
  for (int q = 0; q < vw->world; ++q) {
    for (int kind = 0; kind < 2; ++kind) {
      const unsigned m = kind == 0 ? s.wr_mask : s.wd_mask;
      if (!((m >> q) & 1u)) continue;
      const unsigned long long v = kind == 0 ? wr : wd;
      auto& dq = kind == 0 ? vw->ready[q][me] : vw->done[q][me];
      const VWorld::Ent* hit = nullptr;
      while (!(hit = find(dq, v))) {
        if (vw->aborted) return fail(HZ_ERR_ABORTED, "virtual world aborted");
        if (vw->cv.wait_until(lock, deadline) == std::cv_status::timeout && !find(dq, v)) {
          *reinterpret_cast<volatile unsigned*>(ctx->p2p.abort_host) = 1u;
          return fail(HZ_ERR_ABORTED, std::string("virtual world: rank ") + std::to_string(me) + " timed out waiting for " +
                                          (kind == 0 ? "ready" : "done") + " >= " + std::to_string(v) + " from rank " +
                                          std::to_string(q));
        }
      }
      cudaError_t err = cudaStreamWaitEvent(st, hit->ev->e, 0);
      if (err != cudaSuccess) return cuda_fail(err, "virtual world: cudaStreamWaitEvent");
    }
  }
  return HZ_OK;
}

hz_status vw_signal(hz_ctx* ctx, const SyncArgs& s, cudaStream_t st) {
  if (!(s.sr_mask | s.sd_mask)) return HZ_OK;
  VWorld* vw = ctx->p2p.vw;
  auto ev = std::make_shared<VWorld::Ev>();
  cudaError_t err = cudaEventCreateWithFlags(&ev->e, cudaEventDisableTiming);
  if (err == cudaSuccess) err = cudaEventRecord(ev->e, st);
  if (err != cudaSuccess) return cuda_fail(err, "virtual world: event record");
  const unsigned long long e = ctx->p2p.epoch_host;
  const int me = ctx->rank;
  {
    std::lock_guard<std::mutex> lock(vw->mu);
    for (int q = 0; q < vw->world; ++q) {
      if ((s.sr_mask >> q) & 1u) vw->ready[me][q].push_back(VWorld::Ent{s.sig_ready + e, ev});
      if ((s.sd_mask >> q) & 1u) vw->done[me][q].push_back(VWorld::Ent{s.sig_done + e, ev});
    }
  }
  vw->cv.notify_all();
  return HZ_OK;
}

void vw_abort(hz_ctx* ctx) {
  VWorld* vw = ctx->p2p.vw;
  {
    std::lock_guard<std::mutex> lock(vw->mu);
    vw->aborted = true;
  }
  vw->cv.notify_all();
}

void vw_release(hz_ctx* ctx) {
  VWorld* vw = ctx->p2p.vw;
  bool last = false;
  {
    std::lock_guard<std::mutex> lock(vw->mu);
    last = --vw->refs == 0;
  }
  if (!last) return;
  int cur = 0;
  cudaGetDevice(&cur);
  for (int q = 0; q < vw->world; ++q) {
    cudaSetDevice(vw->devices[q]);
    cudaDeviceSynchronize();
  }
  for (int q = 0; q < vw->world; ++q)
    if (vw->pools[q]) {
      cudaSetDevice(vw->devices[q]);
      cudaFree(vw->pools[q]);
    }
  cudaSetDevice(cur);
  delete vw;
}

}  // namespace hz

extern "C" hz_status hz_init_virtual_ex(hz_ctx** out, int world, int levels, const int* group, const int* devices,
                                        size_t pool_bytes) {
  using namespace hz;
  if (!out) return fail(HZ_ERR_INVALID, "out: NULL");
  if (!group) return fail(HZ_ERR_INVALID, "group: NULL");
  if (levels < 1 || levels > HZ_MAX_LEVELS) return fail(HZ_ERR_INVALID, "levels: must be in [1, 4]");
  int64_t prod = 1;
  for (int l = 0; l < levels; ++l) {
    if (group[l] < 1) return fail(HZ_ERR_INVALID, "group[" + std::to_string(l) + "]: must be >= 1");
    prod *= group[l];
  }
  if (world < 1 || prod != world) return fail(HZ_ERR_INVALID, "group: product must equal world");
  if (world > kMaxWorld) return fail(HZ_ERR_UNSUPPORTED, "virtual world: at most 8 ranks");
  if (!devices) return fail(HZ_ERR_INVALID, "devices: NULL");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  for (int r = 0; r < world; ++r)
    if (devices[r] < 0 || devices[r] >= ndev)
      return fail(HZ_ERR_INVALID, "devices[" + std::to_string(r) + "]: no such CUDA device");
  // ranks on different GPUs read each other's pools directly (same process: peer
  // access instead of IPC)
  for (int a = 0; a < world; ++a)
    for (int b = 0; b < world; ++b) {
      if (devices[a] == devices[b]) continue;
      int can = 0;
      if ((e = cudaDeviceCanAccessPeer(&can, devices[a], devices[b])) != cudaSuccess)
        return cuda_fail(e, "cudaDeviceCanAccessPeer");
      if (!can) return fail(HZ_ERR_UNSUPPORTED, "virtual world: no peer access between the devices of ranks " +
                                                    std::to_string(a) + " and " + std::to_string(b));
      if ((e = cudaSetDevice(devices[a])) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
      e = cudaDeviceEnablePeerAccess(devices[b], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        (void)cudaGetLastError();
      } else if (e != cudaSuccess) {
        return cuda_fail(e, "cudaDeviceEnablePeerAccess");
      }
    }
  for (int r = 0; r < world; ++r) out[r] = nullptr;
  const size_t gran = size_t(2) << 20;
  const size_t total = (kPoolHeader + pool_bytes + gran - 1) / gran * gran;
  VWorld* vw = new VWorld();
  vw->world = world;
  hz_status rc = HZ_OK;
  for (int r = 0; r < world && rc == HZ_OK; ++r) {
    vw->devices[r] = devices[r];
    if ((e = cudaSetDevice(devices[r])) != cudaSuccess || (e = cudaMalloc(&vw->pools[r], total)) != cudaSuccess ||
        (e = cudaMemset(vw->pools[r], 0, kPoolHeader)) != cudaSuccess)
      rc = cuda_fail(e, "virtual world: pool cudaMalloc");
  }
  for (int r = 0; r < world && rc == HZ_OK; ++r) {
    hz_ctx* ctx = new hz_ctx();
    ctx->rank = r;
    ctx->world = world;
    ctx->levels = levels;
    ctx->device = devices[r];
    if ((e = cudaSetDevice(devices[r])) != cudaSuccess) {
      rc = cuda_fail(e, "cudaSetDevice");
      delete ctx;
      break;
    }
    int stride = 1;
    for (int l = 0; l < levels; ++l) {
      ctx->group[l] = group[l];
      ctx->digit[l] = (r / stride) % group[l];
      stride *= group[l];
    }
    auto& P = ctx->p2p;
    P.pool = vw->pools[r];
    P.bytes = total;
    P.used = kPoolHeader;
    for (int q = 0; q < world; ++q) P.peer[q] = vw->pools[q];
    P.vw = vw;
    ++vw->refs;
    out[r] = ctx;
    if ((rc = p2p_alloc_abort(ctx)) != HZ_OK) break;
    P.on = true;
  }
  if (rc != HZ_OK) {
    const std::string msg = hz_last_error();
    if (vw->refs == 0) {   // no context yet: free the world here
      for (int q = 0; q < world; ++q)
        if (vw->pools[q]) cudaFree(vw->pools[q]);
      delete vw;
    } else {               // the last context's finalize frees the pools and the world
      for (int r = 0; r < world; ++r)
        if (out[r]) hz_finalize(out[r]);
    }
    for (int r = 0; r < world; ++r) out[r] = nullptr;
    return fail(rc, msg);
  }
  clear_error();
  return HZ_OK;
}

extern "C" hz_status hz_init_virtual(hz_ctx** out, int world, int levels, const int* group, int cuda_device,
                                     size_t pool_bytes) {
  using namespace hz;
  if (cuda_device < 0) return fail(HZ_ERR_INVALID, "cuda_device: negative");
  if (world < 1 || world > kMaxWorld) return hz_init_virtual_ex(out, world, levels, group, nullptr, pool_bytes);
  int dev[kMaxWorld];
  for (int r = 0; r < world; ++r) dev[r] = cuda_device;
  return hz_init_virtual_ex(out, world, levels, group, dev, pool_bytes);
}
