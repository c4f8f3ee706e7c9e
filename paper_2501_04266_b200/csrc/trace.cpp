// Per-launch device timing of libhz's own work: a CUDA event pair recorded on the
// launching stream around every kernel and every NCCL group (hz_trace_*).
// Events are created up front by hz_trace_begin so that recording inside a timed
// region costs two cudaEventRecord calls per launch and no allocation.
#include <mutex>
#include <vector>

#include "hz_internal.h"

namespace hz {
namespace {

struct Rec {
  const char* kind;
  int level, bits;
  int64_t elems, bytes;
  cudaEvent_t a, b;
  cudaStream_t st;
};

std::mutex g_mu;
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
size_t g_used = 0;

void destroy_pool() {
  for (auto e : g_pool) cudaEventDestroy(e);
  g_pool.clear();
  g_recs.clear();
  g_used = 0;
}

}  // namespace

TraceScope::TraceScope(cudaStream_t st, const char* kind, int level, int bits, int64_t elems,
                       int64_t bytes)
    : active(false), slot(-1), stream(st) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (!g_on || g_used + 2 > g_pool.size()) return;
  Rec r{kind, level, bits, elems, bytes, g_pool[g_used], g_pool[g_used + 1], st};
  g_used += 2;
  if (cudaEventRecord(r.a, st) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  g_recs.push_back(r);
  slot = static_cast<int>(g_recs.size()) - 1;
  active = true;
}

void TraceScope::end() {
  if (!active) return;
  std::lock_guard<std::mutex> lock(g_mu);
  if (slot >= 0 && slot < static_cast<int>(g_recs.size())) {
    if (cudaEventRecord(g_recs[slot].b, stream) != cudaSuccess) cudaGetLastError();
  }
  active = false;
}

TraceScope::~TraceScope() { end(); }

}  // namespace hz

extern "C" {

hz_status hz_trace_begin(int capacity) {
  using namespace hz;
  if (capacity < 1 || capacity > (1 << 20)) return fail(HZ_ERR_INVALID, "capacity: must be in [1, 2^20]");
  std::lock_guard<std::mutex> lock(g_mu);
  destroy_pool();
  g_pool.resize(static_cast<size_t>(capacity) * 2);
  for (auto& e : g_pool) {
    if (cudaEventCreate(&e) != cudaSuccess) {
      cudaGetLastError();
      e = nullptr;
      g_pool.clear();
      return fail(HZ_ERR_CUDA, "hz_trace_begin: cudaEventCreate failed");
    }
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
  int n = 0;
  for (const Rec& r : g_recs) {
    if (n >= max) break;
    float ms = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) {
      cudaGetLastError();
      ms = -1.f;
    }
    out[n].kind = r.kind;
    out[n].level = r.level;
    out[n].bits = r.bits;
    out[n].elems = r.elems;
    out[n].bytes = r.bytes;
    out[n].ms = ms;
    ++n;
  }
  *n_out = max > 0 ? n : static_cast<int>(g_recs.size());
  clear_error();
  return HZ_OK;
}

}  // extern "C"
