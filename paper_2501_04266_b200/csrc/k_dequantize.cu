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
#include "codec.cuh"

namespace hz {
namespace {

using namespace dev;

template <int BITS, typename TO, int U>
__global__ void __launch_bounds__(kThreads) k_dequantize(const __grid_constant__ Pieces pc,
                                                         int64_t nunits, int log2b,
                                                         TO* __restrict__ y,
                                                         const __grid_constant__ SyncArgs sy) {
  sync_wait(sy);
  const int lane = threadIdx.x & 31;
  const int64_t warp = global_warp();
  const int64_t nwarps = num_warps();
  const bool copy_sec = pc.sec_c != nullptr;
  // Pieces interleaved by warp tile (32*U units): consecutive tiles alternate between
  // pieces, so local (HBM) and peer (NVLink) tiles are in flight at the same time
  // instead of one half of the layer after the other.
  const bool inter = pc.n > 1 && (pc.len % (256 * U)) == 0;
  const int64_t tiles_per_piece = pc.len / (256 * U);
  for (int64_t base = warp * 32 * U; base < nunits; base += nwarps * 32 * U) {
    int64_t ub = base;            // first unit of this warp tile in the layer
    int jt = -1;                  // its piece, when interleaved
    if (inter) {
      const int64_t tile = base / (32 * U);
      jt = static_cast<int>(tile % pc.n);
      ub = jt * (pc.len / 8) + (tile / pc.n) * (32 * U);
      (void)tiles_per_piece;
    }
    Codes8<BITS> raw[U];
    float sc[U];
    bool fast = false;
    if constexpr (U == 4) {
      if (log2b == 8 && (inter || (pc.n == 1 && ub + 32 * U <= nunits))) {
        // B = 256, a full tile: its 4 blocks have 4 consecutive scales — one 16-byte
        // (broadcast) load instead of 4 single-scale requests (peer reads are
        // request-bound for small transfers)
        if (!inter) jt = 0;
        const int64_t r0 = ub * 8 - jt * pc.len;
        const bool head = r0 < pc.split && pc.cr[jt] != nullptr;
        const uint8_t* cb = (head ? pc.cr[jt] : pc.c[jt]) + (r0 + lane * 8) * BITS / 8;
        const float4 s4 = __ldg(reinterpret_cast<const float4*>((head ? pc.sr[jt] : pc.s[jt]) + (r0 >> 8)));
#pragma unroll
        for (int u = 0; u < U; ++u) raw[u].load(cb + u * 256 * BITS / 8);
        sc[0] = s4.x;
        sc[1] = s4.y;
        sc[2] = s4.z;
        sc[3] = s4.w;
        fast = true;
      } else if (inter || (pc.n == 1 && ub + 32 * U <= nunits)) {
        // any other block size, a full tile (1024 elements starting at a multiple of
        // 1024): its NS = max(1, 1024/B) scales are consecutive — lane k < NS loads
        // scale k (one request for the tile), every lane takes its unit's scale by
        // shuffle.  (B >= 1024: the tile lies inside one block, NS = 1.)
        if (!inter) jt = 0;
        const int64_t r0 = ub * 8 - jt * pc.len;
        const bool head = r0 < pc.split && pc.cr[jt] != nullptr;
        const uint8_t* cb = (head ? pc.cr[jt] : pc.c[jt]) + (r0 + lane * 8) * BITS / 8;
        const int ns = log2b >= 10 ? 1 : (1024 >> log2b);
        const float mine = __ldg((head ? pc.sr[jt] : pc.s[jt]) + (r0 >> log2b) + (lane < ns ? lane : ns - 1));
#pragma unroll
        for (int u = 0; u < U; ++u) raw[u].load(cb + u * 256 * BITS / 8);
#pragma unroll
        for (int u = 0; u < U; ++u) sc[u] = __shfl_sync(0xffffffffu, mine, (u * 256 + lane * 8) >> log2b);
        fast = true;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t unit = ub + u * 32 + lane;
      if (!fast && unit < nunits) {
        const int64_t e = unit * 8;
        int j = jt;
        if (j < 0) {
          j = 0;
          for (int q = 1; q < pc.n; ++q) j += e >= q * pc.len;   // piece of this unit
        }
        const int64_t r = e - j * pc.len;
        const bool head = r < pc.split && pc.cr[j] != nullptr;   // pushed head: local receive buffer
        raw[u].load((head ? pc.cr[j] : pc.c[j]) + r * BITS / 8);
        sc[u] = __ldg((head ? pc.sr[j] : pc.s[j]) + (r >> log2b));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t unit = ub + u * 32 + lane;
      if (unit < nunits) {
        float c[8], v[8];
        raw[u].decode(c);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __fmul_rn(c[i], sc[u]);
        Out8<TO>::store(y + unit * 8, v);
        if (copy_sec) {
          const int64_t e = unit * 8;
          if (e >= pc.sec_lo && e < pc.sec_hi) {
            raw[u].store(pc.sec_c + (e - pc.sec_lo) * BITS / 8);
            if (((e - pc.sec_lo) & ((int64_t(1) << log2b) - 1)) == 0) pc.sec_s[(e - pc.sec_lo) >> log2b] = sc[u];
          }
        }
      }
    }
  }
  sync_signal(sy);
}

constexpr int kU = 4;   // units in flight per lane (HZ_TUNE deq_u: 2, 4, 8, 16)

template <int BITS, typename TO, int U>
cudaError_t dequantize_u(const Pieces& pc, int64_t nunits, int log2b, void* y, cudaStream_t st,
                         const SyncArgs& sy) {
  auto kern = k_dequantize<BITS, TO, U>;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), (nunits + 32 * U - 1) / (32 * U));
  return launch_k(kern, grid, st, pc, nunits, log2b, static_cast<TO*>(y), sy);
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
