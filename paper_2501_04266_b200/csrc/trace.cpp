// Per-launch device timing of libhz's own work: a CUDA event pair recorded on the
// launching stream around every kernel and every NCCL group (hz_trace_*).
// Events are created up front by hz_trace_begin so that recording inside a timed
// region costs two cudaEventRecord calls per launch and no allocation.
// With HZ_TRACE_STAMPS every libhz kernel also writes %globaltimer stamps into a
// device array (CTA 0 at entry and after its cross-GPU wait, the last CTA to
// finish, and in P2P mode after the flag publication): a per-launch duration
// measured on the device without any extra stream operation (CUDA events
// between dependent launches cost several microseconds each).
#include <mutex>
#include <vector>

#include "hz_internal.h"

namespace hz {
namespace {

struct Rec {
  const char* kind;
  int level, bits;
  int64_t elems, bytes, remote;
  cudaEvent_t a, b;
  cudaStream_t st;
};

// per host thread: the contexts of a virtual world run one per thread and trace
// separately (the mutex only guards against a reader on the same thread's state)
thread_local std::mutex g_mu;
thread_local bool g_on = false;
thread_local std::vector<Rec> g_recs;
thread_local std::vector<cudaEvent_t> g_pool;
thread_local size_t g_used = 0;
thread_local unsigned long long* g_stamps = nullptr;   // device [capacity][8]
thread_local bool g_events = true;
thread_local size_t g_cap = 0;

void destroy_pool() {
  for (auto e : g_pool) cudaEventDestroy(e);
  g_pool.clear();
  g_recs.clear();
  g_used = 0;
  if (g_stamps) cudaFree(g_stamps);
  g_stamps = nullptr;
  g_cap = 0;
}

}  // namespace

TraceScope::TraceScope(cudaStream_t st, const char* kind, int level, int bits, int64_t elems,
                       int64_t bytes, int64_t remote)
    : active(false), slot(-1), stream(st), stamps(nullptr) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (!g_on || g_used + 2 > g_pool.size()) return;
  Rec r{kind, level, bits, elems, bytes, remote, g_pool[g_used], g_pool[g_used + 1], st};
  g_used += 2;
  if (g_events && cudaEventRecord(r.a, st) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  g_recs.push_back(r);
  slot = static_cast<int>(g_recs.size()) - 1;
  if (g_stamps && static_cast<size_t>(slot) < g_cap) stamps = g_stamps + 8 * slot;
  active = true;
}

void TraceScope::end() {
  if (!active) return;
  std::lock_guard<std::mutex> lock(g_mu);
  if (g_events && slot >= 0 && slot < static_cast<int>(g_recs.size())) {
    if (cudaEventRecord(g_recs[slot].b, stream) != cudaSuccess) cudaGetLastError();
  }
  active = false;
}

TraceScope::~TraceScope() { end(); }

}  // namespace hz

extern "C" {

hz_status hz_trace_begin(int capacity, int flags) {
  using namespace hz;
  if (capacity < 1 || capacity > (1 << 20)) return fail(HZ_ERR_INVALID, "capacity: must be in [1, 2^20]");
  if (!(flags & (HZ_TRACE_EVENTS | HZ_TRACE_STAMPS))) return fail(HZ_ERR_INVALID, "flags: no timer selected");
  std::lock_guard<std::mutex> lock(g_mu);
  destroy_pool();
  g_events = (flags & HZ_TRACE_EVENTS) != 0;
  g_pool.resize(static_cast<size_t>(capacity) * 2);
  for (auto& e : g_pool) {
    if (cudaEventCreate(&e) != cudaSuccess) {
      cudaGetLastError();
      e = nullptr;
      g_pool.clear();
      return fail(HZ_ERR_CUDA, "hz_trace_begin: cudaEventCreate failed");
    }
  }
  if (!(flags & HZ_TRACE_STAMPS)) {
    g_stamps = nullptr;
  } else if (cudaMalloc(&g_stamps, sizeof(unsigned long long) * 8 * capacity) != cudaSuccess ||
      cudaMemset(g_stamps, 0, sizeof(unsigned long long) * 8 * capacity) != cudaSuccess) {
    cudaGetLastError();
    g_stamps = nullptr;
  } else {
    g_cap = static_cast<size_t>(capacity);
  }
  g_recs.reserve(capacity);
  g_on = true;
  clear_error();
  return HZ_OK;
}

hz_status hz_trace_end(void) {
  std::lock_guard<std::mutex> lock(hz::g_mu);
  hz::g_on = false;
  hz::clear_error();
  return HZ_OK;
}

hz_status hz_trace_read(hz_trace_rec* out, int max, int* n_out) {
  using namespace hz;
  if (!n_out) return fail(HZ_ERR_INVALID, "n_out: NULL");
  if (max > 0 && !out) return fail(HZ_ERR_INVALID, "out: NULL");
  std::lock_guard<std::mutex> lock(g_mu);
  std::vector<unsigned long long> st;
  const size_t nrec = g_recs.size();
  if (max > 0 && g_stamps && nrec) {
    const size_t cnt = nrec < g_cap ? nrec : g_cap;
    st.resize(8 * cnt);
    cudaDeviceSynchronize();
    if (cudaMemcpy(st.data(), g_stamps, st.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost) !=
        cudaSuccess) {
      cudaGetLastError();
      st.clear();
    }
  }
  int n = 0;
  for (size_t i = 0; i < nrec; ++i) {
    if (n >= max) break;
    const Rec& r = g_recs[i];
    float ms = -1.f;
    if (g_events &&
        (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess)) {
      cudaGetLastError();
      ms = -1.f;
    }
    out[n].kind = r.kind;
    out[n].level = r.level;
    out[n].bits = r.bits;
    out[n].elems = r.elems;
    out[n].bytes = r.bytes;
    out[n].remote_bytes = r.remote;
    out[n].ms = ms;
    out[n].wait_ms = -1.f;
    out[n].work_ms = -1.f;
    out[n].publish_ms = -1.f;
    out[n].stamp_ms = -1.f;
    const unsigned long long* t = st.size() >= 8 * (i + 1) ? &st[8 * i] : nullptr;
    if (t && t[0] && t[1] && t[2] >= t[1]) {
      // duration = entry to the end of the flag publication when the kernel published
      // (t[3]), else to the last CTA's arrival
      const bool pub = t[3] >= t[2] && t[3] != 0;
      out[n].wait_ms = static_cast<float>(t[1] - t[0]) * 1e-6f;
      out[n].work_ms = static_cast<float>(t[2] - t[1]) * 1e-6f;
      out[n].stamp_ms = static_cast<float>((pub ? t[3] : t[2]) - t[0]) * 1e-6f;
      out[n].publish_ms = pub ? static_cast<float>(t[3] - t[2]) * 1e-6f : -1.f;
    }
    ++n;
  }
  *n_out = max > 0 ? n : static_cast<int>(nrec);
  clear_error();
  return HZ_OK;
}

}  // extern "C"
