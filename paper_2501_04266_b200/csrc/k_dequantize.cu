// k_dequantize (A5 forward / A6 backward; oracle O6): codes + fp32 scales ->
// bf16 | fp16 | fp32, x_hat = fl(code * scale), RNE narrowing.  Every rank,
// the owner of a shard included, dequantizes the whole gathered layer from the
// codes (R9), so the layer is bit-identical on all ranks.  Paper: "quantizer and
// dequantizer operators from ZeRO++".
//
// The same kernel is the fused all-gather + dequantize of the NVLink P2P
// transport: the layer is a list of pieces (one per member of the gathering
// group, piece j = elements [j*len, (j+1)*len)), each read straight from the
// owner's IPC-mapped buffer over NVLink (peer loads) or from local HBM, so the
// gathered codes are never materialised.  With one local piece it is a plain
// dequantize.  Optionally the codes of [sec_lo, sec_hi) are copied to the hpZ
// secondary on the way (setting Z, s < w).  In P2P mode the prologue waits for
// the producers' ready flags and the epilogue signals done (codec.cuh).
//
// Elementwise: a unit = 8 consecutive elements (8/4 code bytes in, one 16-byte
// bf16 store out); the lanes of a warp own 32 consecutive units per instruction
// (contiguous spans); each lane keeps U units in flight.
#include "dequantize_loop.cuh"

namespace hz {
namespace {

using namespace dev;

template <int BITS, typename TO, int U>
__global__ void __launch_bounds__(kThreads) k_dequantize(const __grid_constant__ Pieces pc,
                                                         int64_t nunits, int log2b,
                                                         TO* __restrict__ y, int bulk_on,
                                                         const __grid_constant__ SyncArgs sy) {
  __shared__ __align__(128) uint4 stage[kThreads / 32][2 * 256 * sizeof(TO) / 16];
  if (!sync_wait(sy)) return;
  // HZ_TUNE fbd=1: the output by TMA bulk stores.  Off by default since the world-1 carveout
  // (hz_internal.h CarveScope): with it the LSU stores are faster, 27.0 vs 29.0 us per launch
  // (profiles/tma_r02.md, carveout addendum)
  BulkOut bo{stage[threadIdx.x >> 5], 0};
  // (one local piece: the N = 1 dequantize; gathers with peer pieces keep the LSU stores,
  // bulk stores measured neutral-to-slower there)
  const bool bulk = bulk_on && pc.n == 1 && (reinterpret_cast<uintptr_t>(y) & 15u) == 0;
  dequantize_loop<BITS, TO, U>(pc, nunits, log2b, y, global_warp(), num_warps(), 0, INT64_MAX, bulk ? &bo : nullptr);
  if (bulk) bulk_out_finish(threadIdx.x & 31);
  sync_signal(sy);
}

constexpr int kU = 4;   // units in flight per lane (HZ_TUNE deq_u: 2, 4, 8, 16)

template <int BITS, typename TO, int U>
cudaError_t dequantize_u(const Pieces& pc, int64_t nunits, int log2b, void* y, cudaStream_t st,
                         const SyncArgs& sy) {
  auto kern = k_dequantize<BITS, TO, U>;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), (nunits + 32 * U - 1) / (32 * U));
  return launch_k(kern, grid, st, pc, nunits, log2b, static_cast<TO*>(y), tune_param("fbd", 0), sy);
}

template <int BITS, typename TO>
cudaError_t dequantize_t(const Pieces& pc, int64_t n, int block, void* y, cudaStream_t st,
                         const SyncArgs& sy) {
  const int64_t nunits = n / 8;
  int log2b = 0;
  while ((1 << log2b) < block) ++log2b;
  switch (tune_param("deq_u", kU)) {
    case 2: return dequantize_u<BITS, TO, 2>(pc, nunits, log2b, y, st, sy);
    case 8: return dequantize_u<BITS, TO, 8>(pc, nunits, log2b, y, st, sy);
    case 16: return dequantize_u<BITS, TO, 16>(pc, nunits, log2b, y, st, sy);
    default: return dequantize_u<BITS, TO, kU>(pc, nunits, log2b, y, st, sy);
  }
}

template <int BITS>
cudaError_t dequantize_b(const Pieces& pc, int64_t n, int block, void* y, hz_dtype out_dt,
                         cudaStream_t st, const SyncArgs& sy) {
  switch (out_dt) {
    case HZ_F32: return dequantize_t<BITS, float>(pc, n, block, y, st, sy);
    case HZ_BF16: return dequantize_t<BITS, __nv_bfloat16>(pc, n, block, y, st, sy);
    case HZ_F16: return dequantize_t<BITS, __half>(pc, n, block, y, st, sy);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_gather_dequantize(const Pieces& pc, int64_t n, int bits, int block, void* y,
                                     hz_dtype out_dt, cudaStream_t st, const SyncArgs* sync) {
  const SyncArgs sy = sync ? *sync : SyncArgs{};
  if (n == 0 && !sync) return cudaSuccess;
  if (pc.n * pc.len == n && n > 0) {
    const cudaError_t e = tiles_gather(pc, bits, block, y, out_dt, st, sy);
    if (e != cudaErrorNotSupported) return e;
  }
  return bits == 8 ? dequantize_b<8>(pc, n, block, y, out_dt, st, sy)
                   : dequantize_b<4>(pc, n, block, y, out_dt, st, sy);
}

cudaError_t launch_dequantize(const uint8_t* codes, const float* scales, int64_t n, int bits,
                              int block, void* y, hz_dtype out_dt, cudaStream_t st) {
  Pieces pc{};
  pc.c[0] = codes;
  pc.s[0] = scales;
  pc.n = 1;
  pc.len = n;
  return launch_gather_dequantize(pc, n, bits, block, y, out_dt, st, nullptr);
}

}  // namespace hz
