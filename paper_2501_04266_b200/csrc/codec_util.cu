// Grid sizing for the grid-stride codec kernels: SMs x resident CTAs (occupancy
// API, cached per kernel), never more CTAs than there is work for.
#include <atomic>
#include <mutex>
#include <unordered_map>

#include "codec.cuh"

namespace hz {

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 148;
  }
  return cached[dev];
}

namespace {

// per (device, kernel, dynamic shared memory); a kernel with dynamic shared memory above
// the default 48 KB gets the opt-in attribute first (per device)
int resident_ctas(const void* kernel, int dyn_smem) {
  static std::mutex mu;
  struct Key {
    int dev;
    const void* k;
    int smem;
    bool operator==(const Key& o) const { return dev == o.dev && k == o.k && smem == o.smem; }
  };
  struct H {
    size_t operator()(const Key& x) const {
      return std::hash<const void*>()(x.k) ^ (static_cast<size_t>(x.smem) << 8) ^ static_cast<size_t>(x.dev);
    }
  };
  static std::unordered_map<Key, int, H> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  const Key key{dev, kernel, dyn_smem};
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (dyn_smem > 48 * 1024 &&
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem) != cudaSuccess)
    cudaGetLastError();
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, dev::kThreads, dyn_smem) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = 1;
  }
  cache[key] = n;
  return n;
}

}  // namespace

std::atomic<int> g_sm_budget{0};

int64_t grid_for(const void* kernel, int64_t warp_tasks, int dyn_smem) {
  const int64_t per_cta = dev::kThreads / 32;
  const int64_t need = (warp_tasks + per_cta - 1) / per_cta;
  const int budget = g_sm_budget.load(std::memory_order_relaxed);
  const int sms = budget > 0 && budget < sm_count() ? budget : sm_count();
  int64_t cap = static_cast<int64_t>(sms) * resident_ctas(kernel, dyn_smem);
  // HZ_TUNE grid_np=k: non-persistent grids of up to k x the resident capacity
  // (short CTAs the block scheduler can interleave with other streams' kernels)
  static const int np = tune_param("grid_np", 0);
  if (np > 0) cap *= np;
  const int64_t g = need < cap ? need : cap;
  return g < 1 ? 1 : g;
}

}  // namespace hz

#include <cstdlib>
#include <cstring>
#include <string>

namespace hz {

int tune_param(const char* name, int dflt) {
  static const std::string spec = [] {
    const char* e = std::getenv("HZ_TUNE");
    return std::string(e ? e : "");
  }();
  if (spec.empty()) return dflt;
  const std::string key = std::string(name) + "=";
  size_t pos = 0;
  while (pos < spec.size()) {
    size_t end = spec.find(',', pos);
    if (end == std::string::npos) end = spec.size();
    if (spec.compare(pos, key.size(), key) == 0) return std::atoi(spec.c_str() + pos + key.size());
    pos = end + 1;
  }
  return dflt;
}

}  // namespace hz

namespace hz {
namespace {
__global__ void k_epoch_advance(unsigned long long* epoch, unsigned long long span) { *epoch += span; }
}  // namespace

// P2P + CUDA graphs: the last node of a captured step advances the device phase
// epoch, so every replay signals / waits on fresh phase numbers.
cudaError_t launch_epoch_advance(unsigned long long* epoch, unsigned long long span, cudaStream_t st) {
  k_epoch_advance<<<1, 1, 0, st>>>(epoch, span);
  return cudaGetLastError();
}
}  // namespace hz

namespace hz {
namespace {
thread_local int t_carve = -1;
}
int launch_carve() { return t_carve; }
CarveScope::CarveScope(int world) : prev(t_carve) {
  static const int c1 = tune_param("carve1", 100);
  static const int cn = tune_param("carve", -1);
  const int c = world == 1 ? c1 : cn;
  t_carve = c > 100 ? 100 : c;   // percent; negative = the driver default
}
CarveScope::~CarveScope() { t_carve = prev; }

// Off by default: measured on B200 (profiles/bench_r01.md) PDL left the multi-GPU
// step unchanged and made the N = 1 step 7 % slower (the fused round trip 51 -> 56 µs).
bool pdl_enabled() {
  static const bool on = tune_param("pdl", 0) != 0;
  return on;
}
}  // namespace hz

extern "C" hz_status hz_set_sm_budget(int sms) {
  if (sms < 0) return hz::fail(HZ_ERR_INVALID, "sms: negative");
  hz::g_sm_budget.store(sms, std::memory_order_relaxed);
  hz::clear_error();
  return HZ_OK;
}
