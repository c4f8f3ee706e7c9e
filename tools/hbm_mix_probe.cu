// HBM read:write mix probe (tool, not product): the bandwidth a plain streaming
// kernel reaches on this B200 for the byte mixes of the libhz kernels, at their
// size (50.4 M elements, the GPT-1.3B layer), so their roofline fractions can be
// read against the same mix instead of the 1:1 copy of MEASURED_PEAKS.json.
//
// Per element the kernel reads RB bytes from one array and writes WB bytes spread
// over up to two arrays (16-byte vector accesses, grid-stride, SMs x 8 CTAs of 256),
// CUDA events over 20 launches rotating over 4 buffer sets (> L2).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_mix_probe tools/hbm_mix_probe.cu && ./hbm_mix_probe
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

// one "unit" = 16 elements: reads RB uint4 (RB bytes per element), writes W1 + W2
// uint4; structure of arrays (stream k at k * units), so every warp access is one
// contiguous 512-byte span
template <int RB, int W1, int W2>
__global__ void __launch_bounds__(256) mix_k(const uint4* __restrict__ in, uint4* __restrict__ o1,
                                             uint4* __restrict__ o2, long units) {
  constexpr int RV = RB, V1 = W1, V2 = W2;
  const long tid = blockIdx.x * 256L + threadIdx.x;
  const long nth = gridDim.x * 256L;
  for (long u = tid; u < units; u += nth) {
    uint4 r[RV > 0 ? RV : 1];
    unsigned acc = 0;
#pragma unroll
    for (int k = 0; k < RV; ++k) {
      r[k] = in[k * units + u];
      acc ^= r[k].x ^ r[k].y ^ r[k].z ^ r[k].w;
    }
#pragma unroll
    for (int k = 0; k < V1; ++k) o1[k * units + u] = make_uint4(acc, acc + k, r[0].y, r[0].z);
#pragma unroll
    for (int k = 0; k < V2; ++k) o2[k * units + u] = make_uint4(acc + 1, acc ^ k, r[0].w, r[0].x);
  }
}

template <int RB, int W1, int W2>
void run(const char* what, long n, int sms) {
  const long units = n / 16;
  const int sets = 4;
  uint4 *in[sets], *o1[sets], *o2[sets];
  for (int s = 0; s < sets; ++s) {
    CK(cudaMalloc(&in[s], n * RB));
    CK(cudaMalloc(&o1[s], n * W1 + 16));
    CK(cudaMalloc(&o2[s], n * W2 + 16));
    CK(cudaMemset(in[s], 1, n * RB));
  }
  const int grid = sms * 8;
  for (int s = 0; s < sets; ++s) mix_k<RB, W1, W2><<<grid, 256>>>(in[s], o1[s], o2[s], units);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int iters = 20;
  CK(cudaEventRecord(a));
  for (int i = 0; i < iters; ++i) mix_k<RB, W1, W2><<<grid, 256>>>(in[i % sets], o1[i % sets], o2[i % sets], units);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  CK(cudaGetLastError());
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  ms /= iters;
  const double bytes = double(n) * (RB + W1 + W2);
  printf("%-44s read %d B + write %d B per element: %7.1f us  %7.1f GB/s\n", what, RB, W1 + W2, ms * 1e3,
         bytes / (ms * 1e-3) / 1e9);
  for (int s = 0; s < sets; ++s) {
    CK(cudaFree(in[s]));
    CK(cudaFree(o1[s]));
    CK(cudaFree(o2[s]));
  }
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long n = 50358272;   // GPT-1.3B layer, padded
  run<2, 2, 0>("1:1 copy (bf16 -> bf16)", n, sms);
  run<4, 4, 0>("1:1 copy (fp32 -> fp32)", n, sms);
  run<2, 2, 1>("fwd round trip mix (bf16 -> bf16 + int8)", n, sms);
  run<2, 4, 0>("qgZ round trip mix (bf16 -> fp32)", n, sms);
  run<1, 2, 0>("dequantize mix (int8 -> bf16)", n, sms);
  run<2, 1, 0>("quantize mix (bf16 -> int8)", n, sms);
  run<2, 2, 0>("1:1 copy again", n, sms);
  printf("done\n");
  return 0;
}
