// The gather+dequantize loop of k_dequantize (see k_dequantize.cu), shared with the
// dual kernel of k_quantize.cu (k_gather_quantize): warp `warp` of `nwarps` processes
// its grid-stride share of the layer.  Internal header.
#pragma once

#include "codec.cuh"

namespace hz {
namespace dev {

// Optional TMA stores of the output (k_dequantize): a full warp step's 256 outputs land in
// one of this warp's two shared-memory buffers (256 * sizeof(TO) bytes each) and lane 0
// bulk-stores the contiguous span; the buffer is reused after its store has read it.
struct BulkOut {
  uint4* stage;   // 2 buffers of 256 * sizeof(TO) bytes
  int buf;
};
template <typename TO>
__device__ __forceinline__ void bulk_out_step(BulkOut& bo, TO* dst, int lane, const float (&v)[8]) {
  constexpr int SPAN = 256 * static_cast<int>(sizeof(TO));
  TO* st = reinterpret_cast<TO*>(reinterpret_cast<char*>(bo.stage) + bo.buf * SPAN);
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
  __syncwarp();
  Out8<TO>::store(st + lane * 8, v);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(static_cast<uint32_t>(__cvta_generic_to_shared(st))), "n"(SPAN)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  bo.buf ^= 1;
}
__device__ __forceinline__ void bulk_out_finish(int lane) {
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncwarp();
}

// Warp tiles [tile0, tile1) of the layer only (32*U units each; default: all of them).
template <int BITS, typename TO, int U>
__device__ __forceinline__ void dequantize_loop(const Pieces& pc, int64_t nunits, int log2b, TO* __restrict__ y,
                                                int64_t warp, int64_t nwarps, int64_t tile0 = 0,
                                                int64_t tile1 = INT64_MAX, BulkOut* bo = nullptr) {
  const int lane = threadIdx.x & 31;
  const bool copy_sec = pc.sec_c != nullptr;
  // Pieces interleaved by warp tile (32*U units): consecutive tiles alternate between
  // pieces, so local (HBM) and peer (NVLink) tiles are in flight at the same time
  // instead of one half of the layer after the other.
  const bool inter = pc.n > 1 && (pc.len % (256 * U)) == 0;
  const int64_t tiles_per_piece = pc.len / (256 * U);
  const int64_t end = tile1 < (nunits + 32 * U - 1) / (32 * U) ? tile1 * 32 * U : nunits;
  for (int64_t base = (tile0 + warp) * 32 * U; base < end; base += nwarps * 32 * U) {
    int64_t ub = base;            // first unit of this warp tile in the layer
    int jt = -1;                  // its piece, when interleaved
    if (inter) {
      // tile -> (piece, tile of that piece): for each q = tile / n the n tiles go to the n
      // pieces, rotated by one piece per grid-stride pass (q / (nwarps / n)), so a warp's
      // successive tiles alternate between the local piece and the peers' pieces.  (With
      // piece = tile % n and nwarps a multiple of n, every warp would read the same piece
      // on every pass: half the warps all-NVLink, half all-HBM, the launch ending with
      // the slower half.)
      const int64_t tile = base / (32 * U);
      const int64_t q = tile / pc.n;
      const int64_t rot = nwarps >= pc.n ? q / (nwarps / pc.n) : 0;
      jt = static_cast<int>((tile % pc.n + rot) % pc.n);
      ub = jt * (pc.len / 8) + q * (32 * U);
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
        const uint8_t* cb = pc.c[jt] + (r0 + lane * 8) * BITS / 8;
        const float4 s4 = HZ_PEER_LD(reinterpret_cast<const float4*>(pc.s[jt] + (r0 >> 8)));
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
        const uint8_t* cb = pc.c[jt] + (r0 + lane * 8) * BITS / 8;
        const int ns = log2b >= 10 ? 1 : (1024 >> log2b);
        const float mine = HZ_PEER_LD(pc.s[jt] + (r0 >> log2b) + (lane < ns ? lane : ns - 1));
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
        raw[u].load(pc.c[j] + r * BITS / 8);
        sc[u] = HZ_PEER_LD(pc.s[j] + (r >> log2b));
      }
    }
    if (bo && fast && !copy_sec) {   // a full tile: 32*U contiguous units, TMA stores
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float c[8], v[8];
        raw[u].decode(c);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __fmul_rn(c[i], sc[u]);
        bulk_out_step<TO>(*bo, y + (ub + u * 32) * 8, lane, v);
      }
      continue;
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
}

}  // namespace dev
}  // namespace hz
