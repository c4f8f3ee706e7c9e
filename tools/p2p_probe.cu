// NVLink peer-access probe (tool, not product): one process, two GPUs with peer
// access enabled.  Measures, with CUDA events, the bandwidth of SM-driven peer
// reads / writes at several per-lane widths and loads-in-flight, one-way and
// both GPUs at once, next to the copy-engine peer copy.  Informs the P2P
// transport design.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_probe tools/p2p_probe.cu && ./p2p_probe
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

// read `n` vectors of V from src, write them to dst (src and/or dst may be peer memory)
template <typename V, int U>
__global__ void __launch_bounds__(256) copy_k(const V* __restrict__ src, V* __restrict__ dst, long n) {
  const long tid = blockIdx.x * 256L + threadIdx.x;
  const long nth = gridDim.x * 256L;
  for (long base = tid; base < n; base += nth * U) {
    V r[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * nth < n) r[u] = src[base + u * nth];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * nth < n) dst[base + u * nth] = r[u];
  }
}

template <typename V, int U>
float run(int dev_exec, const void* src, void* dst, size_t bytes, int iters, int grid, cudaStream_t st) {
  CK(cudaSetDevice(dev_exec));
  const long n = bytes / sizeof(V);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  copy_k<V, U><<<grid, 256, 0, st>>>((const V*)src, (V*)dst, n);
  CK(cudaEventRecord(a, st));
  for (int i = 0; i < iters; ++i) copy_k<V, U><<<grid, 256, 0, st>>>((const V*)src, (V*)dst, n);
  CK(cudaEventRecord(b, st));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / iters;
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, 0, 1));
  printf("can access peer 0->1: %d\n", can);
  const size_t bytes = size_t(64) << 20;   // 64 MB per buffer
  void *l0, *l0b, *l1, *l1b;
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&l0, bytes));
  CK(cudaMalloc(&l0b, bytes));
  cudaStream_t s0, s1;
  CK(cudaStreamCreate(&s0));
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaMalloc(&l1, bytes));
  CK(cudaMalloc(&l1b, bytes));
  CK(cudaStreamCreate(&s1));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int iters = 20;
  struct Cfg { const char* name; int grid_mult; };
  for (int gm : {2, 4, 8}) {
    const int grid = sms * gm;
    // local copy (GPU0)
    float t = run<uint4, 4>(0, l0, l0b, bytes, iters, grid, s0);
    printf("grid=%d local copy uint4 U4        : %7.1f GB/s (rd+wr)\n", grid, 2 * bytes / t / 1e6);
    // peer read: GPU0 reads GPU1 memory, writes local
    t = run<uint2, 4>(0, l1, l0b, bytes, iters, grid, s0);
    printf("grid=%d peer read  uint2 U4        : %7.1f GB/s (remote bytes)\n", grid, bytes / t / 1e6);
    t = run<uint4, 4>(0, l1, l0b, bytes, iters, grid, s0);
    printf("grid=%d peer read  uint4 U4        : %7.1f GB/s\n", grid, bytes / t / 1e6);
    t = run<uint4, 8>(0, l1, l0b, bytes, iters, grid, s0);
    printf("grid=%d peer read  uint4 U8        : %7.1f GB/s\n", grid, bytes / t / 1e6);
    t = run<unsigned short, 4>(0, l1, l0b, bytes / 8, iters, grid, s0);
    printf("grid=%d peer read  u16   U4 (1/8 sz): %7.1f GB/s\n", grid, bytes / 8 / t / 1e6);
    // peer write: GPU0 reads local, writes GPU1 memory
    t = run<uint4, 4>(0, l0, l1b, bytes, iters, grid, s0);
    printf("grid=%d peer write uint4 U4        : %7.1f GB/s\n", grid, bytes / t / 1e6);
    t = run<uint2, 4>(0, l0, l1b, bytes, iters, grid, s0);
    printf("grid=%d peer write uint2 U4        : %7.1f GB/s\n", grid, bytes / t / 1e6);
  }
  // both directions at once: GPU0 reads GPU1 and GPU1 reads GPU0
  {
    const int grid = sms * 4;
    cudaEvent_t a0, b0, a1, b1;
    CK(cudaSetDevice(0));
    CK(cudaEventCreate(&a0));
    CK(cudaEventCreate(&b0));
    CK(cudaSetDevice(1));
    CK(cudaEventCreate(&a1));
    CK(cudaEventCreate(&b1));
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaSetDevice(0));
      CK(cudaEventRecord(a0, s0));
      for (int i = 0; i < iters; ++i) copy_k<uint4, 4><<<grid, 256, 0, s0>>>((const uint4*)l1, (uint4*)l0b, bytes / 16);
      CK(cudaEventRecord(b0, s0));
      CK(cudaSetDevice(1));
      CK(cudaEventRecord(a1, s1));
      for (int i = 0; i < iters; ++i) copy_k<uint4, 4><<<grid, 256, 0, s1>>>((const uint4*)l0, (uint4*)l1b, bytes / 16);
      CK(cudaEventRecord(b1, s1));
      CK(cudaEventSynchronize(b0));
      CK(cudaEventSynchronize(b1));
    }
    float m0, m1;
    CK(cudaEventElapsedTime(&m0, a0, b0));
    CK(cudaEventElapsedTime(&m1, a1, b1));
    printf("bidirectional peer read uint4: GPU0 %7.1f GB/s  GPU1 %7.1f GB/s\n", bytes * iters / m0 / 1e6,
           bytes * iters / m1 / 1e6);
  }
  // copy engine
  {
    CK(cudaSetDevice(0));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaMemcpyPeerAsync(l0b, 0, l1, 1, bytes, s0));
    CK(cudaEventRecord(a, s0));
    for (int i = 0; i < iters; ++i) CK(cudaMemcpyPeerAsync(l0b, 0, l1, 1, bytes, s0));
    CK(cudaEventRecord(b, s0));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("cudaMemcpyPeerAsync 1->0          : %7.1f GB/s\n", bytes * iters / ms / 1e6);
  }
  printf("done\n");
  return 0;
}
