// NVLink peer-read probe at SMALL grids (tool, not product): how many CTAs does a
// peer read need when the rest of the GPU is busy with GEMMs?  Compares, per grid
// size G, (a) plain vectorised loads (256 or 1024 threads, 8 x 16 B in flight per
// thread) with (b) TMA bulk copies (cp.async.bulk global -> shared, mbarrier
// complete_tx) of C-byte chunks into an S-stage shared-memory ring, drained by the
// CTA's threads into local HBM.  One process, two GPUs with peer access; CUDA
// events; 64 MB per transfer.  Informs the low-footprint transport.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_probe tools/bulk_probe.cu && ./bulk_probe
#include <cstdint>
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

template <int T, int U>
__global__ void __launch_bounds__(T) load_k(const uint4* __restrict__ src, uint4* __restrict__ dst, long n) {
  const long tid = blockIdx.x * long(T) + threadIdx.x;
  const long nth = gridDim.x * long(T);
  for (long base = tid; base < n; base += nth * U) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * nth < n) r[u] = src[base + u * nth];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * nth < n) dst[base + u * nth] = r[u];
  }
}

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// chunks of C bytes; chunk k of this CTA = blockIdx.x + j * gridDim.x
template <int T>
__global__ void __launch_bounds__(T) bulk_k(const char* __restrict__ src, char* __restrict__ dst, long nchunks, int C,
                                          int S) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[16];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long mine = nchunks > blockIdx.x ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto issue = [&](long j) {
    const long k = blockIdx.x + j * gridDim.x;
    const int s = j % S;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(C) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa(smem + (size_t)s * C)),
                 "l"(src + k * C), "r"(C), "r"(sa(&bar[s]))
                 : "memory");
  };
  if (tid == 0)
    for (long j = 0; j < S && j < mine; ++j) issue(j);
  for (long j = 0; j < mine; ++j) {
    const int s = j % S;
    const uint32_t par = (j / S) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(sa(&bar[s])), "r"(par)
                   : "memory");
    const uint4* in = reinterpret_cast<const uint4*>(smem + (size_t)s * C);
    uint4* out = reinterpret_cast<uint4*>(dst + (blockIdx.x + j * gridDim.x) * C);
    for (int i = tid; i < C / 16; i += T) out[i] = in[i];
    __syncthreads();
    if (tid == 0 && j + S < mine) issue(j + S);
  }
}

template <typename F>
float timeit(int dev, cudaStream_t st, int iters, F f) {
  CK(cudaSetDevice(dev));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaEventRecord(a, st));
  for (int i = 0; i < iters; ++i) f();
  CK(cudaEventRecord(b, st));
  CK(cudaEventSynchronize(b));
  CK(cudaGetLastError());
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
  const size_t bytes = size_t(64) << 20;
  void *l0, *l0b, *l1;
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&l0, bytes));
  CK(cudaMalloc(&l0b, bytes));
  cudaStream_t s0;
  CK(cudaStreamCreate(&s0));
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaMalloc(&l1, bytes));
  CK(cudaMemset(l1, 1, bytes));
  CK(cudaSetDevice(0));
  CK(cudaFuncSetAttribute(bulk_k<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(bulk_k<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int iters = 10;
  for (int G : {4, 8, 16, 24, 32, 48, 64, 148}) {
    float t1 = timeit(0, s0, iters, [&] {
      load_k<256, 8><<<G, 256, 0, s0>>>((const uint4*)l1, (uint4*)l0b, bytes / 16);
    });
    float t2 = timeit(0, s0, iters, [&] {
      load_k<1024, 8><<<G, 1024, 0, s0>>>((const uint4*)l1, (uint4*)l0b, bytes / 16);
    });
    printf("G=%3d peer read loads  256x8x16B: %6.1f GB/s   1024x8x16B: %6.1f GB/s\n", G, bytes / t1 / 1e6,
           bytes / t2 / 1e6);
    for (int C : {16384, 32768, 49152}) {
      const int S = (192 * 1024) / C;
      float t3 = timeit(0, s0, iters, [&] {
        bulk_k<256><<<G, 256, (size_t)S * C, s0>>>((const char*)l1, (char*)l0b, bytes / C, C, S);
      });
      float t4 = timeit(0, s0, iters, [&] {
        bulk_k<512><<<G, 512, (size_t)S * C, s0>>>((const char*)l1, (char*)l0b, bytes / C, C, S);
      });
      printf("G=%3d peer read bulk C=%5d S=%2d: 256 thr %6.1f GB/s   512 thr %6.1f GB/s\n", G, C, S,
             bytes / t3 / 1e6, bytes / t4 / 1e6);
    }
    // local HBM copy through the bulk ring (same kernel, local source)
    float t5 = timeit(0, s0, iters, [&] {
      bulk_k<512><<<G, 512, (size_t)4 * 49152, s0>>>((const char*)l0, (char*)l0b, bytes / 49152, 49152, 4);
    });
    printf("G=%3d local copy bulk C=49152 S=4 512 thr: %6.1f GB/s (read)\n", G, bytes / t5 / 1e6);
  }
  // both directions at once: GPU0 pulls from GPU1 while GPU1 pulls from GPU0
  {
    void* l1b;
    cudaStream_t s1;
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&l1b, bytes));
    CK(cudaStreamCreate(&s1));
    CK(cudaFuncSetAttribute(bulk_k<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(bulk_k<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    cudaEvent_t a0, b0, a1, b1;
    CK(cudaEventCreate(&a1));
    CK(cudaEventCreate(&b1));
    CK(cudaSetDevice(0));
    CK(cudaEventCreate(&a0));
    CK(cudaEventCreate(&b0));
    for (int mode = 0; mode < 3; ++mode) {
      for (int G : {32, 74, 148, 296}) {
        float m0 = 0, m1 = 0;
        for (int rep = 0; rep < 2; ++rep) {
          for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            cudaStream_t st = d ? s1 : s0;
            const char* src = (const char*)(d ? l0 : l1);
            char* dst = (char*)(d ? l1b : l0b);
            CK(cudaEventRecord(d ? a1 : a0, st));
            for (int i = 0; i < iters; ++i) {
              if (mode == 0)
                load_k<256, 8><<<G * 4, 256, 0, st>>>((const uint4*)src, (uint4*)dst, bytes / 16);
              else if (mode == 1)
                bulk_k<256><<<G, 256, 4 * 49152, st>>>(src, dst, bytes / 49152, 49152, 4);
              else
                bulk_k<512><<<G, 512, 6 * 32768, st>>>(src, dst, bytes / 32768, 32768, 6);
            }
            CK(cudaEventRecord(d ? b1 : b0, st));
          }
          CK(cudaEventSynchronize(b0));
          CK(cudaEventSynchronize(b1));
          CK(cudaEventElapsedTime(&m0, a0, b0));
          CK(cudaEventElapsedTime(&m1, a1, b1));
        }
        const char* nm[3] = {"loads 256x8x16B (4 CTAs per G)", "bulk C=48K S=4 256 thr", "bulk C=32K S=6 512 thr"};
        printf("bidirectional %-32s G=%3d: GPU0 %6.1f GB/s  GPU1 %6.1f GB/s\n", nm[mode], G,
               bytes * iters / m0 / 1e6, bytes * iters / m1 / 1e6);
      }
    }
    CK(cudaSetDevice(0));
  }
  // verify last bulk copy from peer
  CK(cudaSetDevice(0));
  bulk_k<256><<<8, 256, 4 * 32768, s0>>>((const char*)l1, (char*)l0b, bytes / 32768, 32768, 4);
  CK(cudaStreamSynchronize(s0));
  unsigned char h[64];
  CK(cudaMemcpy(h, (char*)l0b + bytes - 64, 64, cudaMemcpyDeviceToHost));
  int ok = 1;
  for (int i = 0; i < 64; ++i) ok &= h[i] == 1;
  printf("verify: %s\ndone\n", ok ? "ok" : "MISMATCH");
  return 0;
}
