// TMA streaming probe (tool, not product): the HBM bandwidth of a streaming kernel whose
// loads AND stores are bulk copies (cp.async.bulk global->shared on an mbarrier ring,
// cp.async.bulk shared->global in bulk groups), for the read:write byte mixes of the
// libhz kernels, against the LSU (ld/st.global) kernel of tools/hbm_mix_probe.cu.  The
// question it answers: with 64-register kernels limited to 32 warps per SM, is a TMA
// pipeline (in-flight bytes held in shared memory, not in registers / L1) faster for the
// write-heavy mixes?
//
// Per tile of TE elements a CTA bulk-loads RB*TE bytes into an input stage (S_IN stages),
// every thread transforms 16-byte chunks into an output buffer (2 buffers) and thread 0
// bulk-stores WB*TE bytes.  SMs x C CTAs of 256 threads, tiles grid-strided; CUDA events
// over 20 launches rotating over 4 buffer sets (> L2).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_mix_probe tools/tma_mix_probe.cu && ./tma_mix_probe
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

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int RB, int WB>
__global__ void __launch_bounds__(256) tma_k(const char* __restrict__ in, char* __restrict__ out, long ntiles, int te,
                                             int s_in) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[8];
  const int ib = RB * te, ob = WB * te;
  char* ibuf = smem;
  char* obuf = smem + s_in * ib;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < s_in; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long mine = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto issue = [&](long j) {
    const long t = blockIdx.x + j * gridDim.x;
    const int s = j % s_in;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(ib) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa(ibuf + s * ib)),
                 "l"(in + t * ib), "r"(ib), "r"(sa(&bar[s]))
                 : "memory");
  };
  if (tid == 0)
    for (long j = 0; j < s_in && j < mine; ++j) issue(j);
  for (long j = 0; j < mine; ++j) {
    const int s = j % s_in;
    const uint32_t par = (j / s_in) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(sa(&bar[s])), "r"(par)
                   : "memory");
    // the output buffer j % 2 was last stored two tiles ago: its bulk store must have read it
    if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    const uint4* src = reinterpret_cast<const uint4*>(ibuf + s * ib);
    uint4* dst = reinterpret_cast<uint4*>(obuf + (j & 1) * ob);
    // each output chunk k derives from input chunk k * RB / WB (touches every input byte)
    for (int k = tid; k < ob / 16; k += 256) {
      const uint4 a = src[(long(k) * RB / WB) % (ib / 16)];
      dst[k] = make_uint4(a.x ^ k, a.y, a.z + 1, a.w);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      const long t = blockIdx.x + j * gridDim.x;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + t * ob), "r"(sa(dst)),
                   "r"(ob)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (j + s_in < mine) {   // input stage s fully consumed (barrier above)
        asm volatile("fence.proxy.async;" ::: "memory");
        issue(j + s_in);
      }
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Hybrid: ld.global loads (registers, 32 warps per SM) and per-warp bulk STORES — each
// warp writes its output span to its own shared-memory buffer (double-buffered) and lane 0
// issues one cp.async.bulk shared -> global per span; no CTA barrier anywhere.  16
// elements per lane per iteration (U units of 16 B input per lane).
template <int RB, int WB, int U>
__global__ void __launch_bounds__(256) hyb_k(const uint4* __restrict__ in, char* __restrict__ out, long units) {
  extern __shared__ __align__(128) char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int SPAN = 32 * U * 16 * WB / RB;            // output bytes per warp iteration
  char* buf = smem + w * 2 * SPAN;
  const long gw = (blockIdx.x * 256L + threadIdx.x) >> 5, nw = (gridDim.x * 256L) >> 5;
  int it = 0;
  for (long base = gw * 32 * U; base < units; base += nw * 32 * U, ++it) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = in[base + u * 32 + lane];
    char* b = buf + (it & 1) * SPAN;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    uint4* o = reinterpret_cast<uint4*>(b);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < WB / RB; ++k) o[(u * (WB / RB) + k) * 32 + lane] = make_uint4(r[u].x ^ k, r[u].y, r[u].z + 1, r[u].w);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + base * 16 * WB / RB),
                   "r"(sa(b)), "r"(SPAN)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int RB, int WB, int U>
void run_hyb(const char* what, long n, int sms, int cpb) {
  const long units = n * RB / 16;
  const int sets = 4;
  char *in[sets], *out[sets];
  for (int s = 0; s < sets; ++s) {
    CK(cudaMalloc(&in[s], n * RB));
    CK(cudaMalloc(&out[s], n * WB));
    CK(cudaMemset(in[s], 1, n * RB));
  }
  const int smem = 8 * 2 * (32 * U * 16 * WB / RB);
  CK(cudaFuncSetAttribute(hyb_k<RB, WB, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hyb_k<RB, WB, U>, 256, smem));
  const int c = cpb < occ ? cpb : occ;
  const int grid = sms * (c > 0 ? c : 1);
  for (int s = 0; s < sets; ++s) hyb_k<RB, WB, U><<<grid, 256, smem>>>((const uint4*)in[s], out[s], units);
  CK(cudaGetLastError());
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int iters = 20;
  CK(cudaEventRecord(a));
  for (int i = 0; i < iters; ++i) hyb_k<RB, WB, U><<<grid, 256, smem>>>((const uint4*)in[i % sets], out[i % sets], units);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  CK(cudaGetLastError());
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  ms /= iters;
  const double bytes = double(n) * (RB + WB);
  printf("HYB %-36s U=%d ctas/SM=%d (smem %6d): %7.1f us  %7.1f GB/s\n", what, U, c, smem, ms * 1e3,
         bytes / (ms * 1e-3) / 1e9);
  for (int s = 0; s < sets; ++s) {
    CK(cudaFree(in[s]));
    CK(cudaFree(out[s]));
  }
}

template <int RB, int WB>
void run(const char* what, long n, int sms, int te, int s_in, int cpb) {
  const long ntiles = n / te;
  const int sets = 4;
  char *in[sets], *out[sets];
  for (int s = 0; s < sets; ++s) {
    CK(cudaMalloc(&in[s], n * RB));
    CK(cudaMalloc(&out[s], n * WB));
    CK(cudaMemset(in[s], 1, n * RB));
  }
  const int smem = s_in * RB * te + 2 * WB * te;
  CK(cudaFuncSetAttribute(tma_k<RB, WB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tma_k<RB, WB>, 256, smem));
  const int c = cpb < occ ? cpb : occ;
  const int grid = sms * (c > 0 ? c : 1);
  for (int s = 0; s < sets; ++s) tma_k<RB, WB><<<grid, 256, smem>>>(in[s], out[s], ntiles, te, s_in);
  CK(cudaGetLastError());
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int iters = 20;
  CK(cudaEventRecord(a));
  for (int i = 0; i < iters; ++i) tma_k<RB, WB><<<grid, 256, smem>>>(in[i % sets], out[i % sets], ntiles, te, s_in);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  CK(cudaGetLastError());
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  ms /= iters;
  const double bytes = double(n) * (RB + WB);
  printf("TMA %-36s te=%5d s_in=%d ctas/SM=%d (smem %6d): %7.1f us  %7.1f GB/s\n", what, te, s_in, c, smem, ms * 1e3,
         bytes / (ms * 1e-3) / 1e9);
  for (int s = 0; s < sets; ++s) {
    CK(cudaFree(in[s]));
    CK(cudaFree(out[s]));
  }
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long n = 50364416;   // GPT-1.3B layer, padded (multiple of 8192)
  if (getenv("HYB")) {
    for (int cpb : {2, 3, 4, 6, 8}) {
      run_hyb<2, 4, 2>("qgZ round trip mix (bf16 -> fp32)", n, sms, cpb);
      run_hyb<2, 4, 4>("qgZ round trip mix (bf16 -> fp32)", n, sms, cpb);
      run_hyb<1, 2, 2>("dequantize mix (int8 -> bf16)", n, sms, cpb);
      run_hyb<1, 2, 4>("dequantize mix (int8 -> bf16)", n, sms, cpb);
      run_hyb<2, 2, 2>("1:1 copy (bf16 -> bf16)", n, sms, cpb);
      run_hyb<2, 2, 4>("1:1 copy (bf16 -> bf16)", n, sms, cpb);
    }
    printf("done\n");
    return 0;
  }
  for (int te : {2048, 4096, 8192}) {
    for (int s_in : {2, 3, 4}) {
      for (int cpb : {2, 4}) {
        run<2, 2>("1:1 copy (bf16 -> bf16)", n, sms, te, s_in, cpb);
        run<2, 3>("fwd round trip mix (bf16 -> bf16 + int8)", n, sms, te, s_in, cpb);
        run<1, 2>("dequantize mix (int8 -> bf16)", n, sms, te, s_in, cpb);
        run<2, 1>("quantize mix (bf16 -> int8)", n, sms, te, s_in, cpb);
        run<2, 4>("qgZ round trip mix (bf16 -> fp32)", n, sms, te, s_in, cpb);
      }
    }
  }
  printf("done\n");
  return 0;
}
