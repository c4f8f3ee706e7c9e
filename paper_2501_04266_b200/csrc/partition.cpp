// Partition / ownership map (O1-O3): Table IV, the dependency rule
// N >= N_os >= N_g >= N_w, primary weights over 2 GCDs.
//
// Hierarchy g = (g_1..g_L), innermost first.  Rank digits (node-major):
//   r = sum_l d_l * prod_{k<l} g_k.
// Padding: Np = ceil(n / (W*4*B)) * W*4*B, so every level chunk is a whole
// number of blocks and every chunk's fp32 scale slice is 16-byte aligned.
// Digit-reversed ranges: off_0 = 0, len_0 = Np, len_l = len_{l-1}/g_l,
// off_l = off_{l-1} + d_l*len_l.  Each level's exchange group therefore owns the
// consecutive pieces of its common range_{l-1} in ascending digit order, so
// every all-gather output and every reduce-scatter chunk is contiguous.
#include <string>

#include "hz_internal.h"

namespace hz {

hz_status partition(int rank, int levels, const int* group, int64_t numel, int block, int w,
                    int s, int gl, hz_partition_t* out) {
  if (!out) return fail(HZ_ERR_INVALID, "out: NULL");
  if (levels < 1 || levels > HZ_MAX_LEVELS)
    return fail(HZ_ERR_INVALID, "levels: must be in [1, " + std::to_string(HZ_MAX_LEVELS) + "]");
  if (!group) return fail(HZ_ERR_INVALID, "group: NULL");
  int64_t world = 1;
  for (int l = 0; l < levels; ++l) {
    if (group[l] < 1 || group[l] > 1024)
      return fail(HZ_ERR_INVALID, "group[" + std::to_string(l) + "]: must be in [1, 1024]");
    world *= group[l];
  }
  if (world > (1 << 20)) return fail(HZ_ERR_INVALID, "group: world too large");
  if (rank < 0 || rank >= world)
    return fail(HZ_ERR_INVALID, "rank: must be in [0, prod(group))");
  if (numel < 0) return fail(HZ_ERR_INVALID, "numel: negative");
  if (!block_ok(block)) return fail(HZ_ERR_INVALID, "block: must be a power of two in [32, 2048]");
  if (w < 0 || w > levels) return fail(HZ_ERR_INVALID, "w: must be in [0, levels]");
  if (s < 0 || s > levels) return fail(HZ_ERR_INVALID, "s: must be in [0, levels]");
  if (gl < 0 || gl > levels) return fail(HZ_ERR_INVALID, "gl: must be in [0, levels]");

  hz_partition_t p{};
  p.numel = numel;
  const int64_t unit = world * 4 * static_cast<int64_t>(block);
  p.padded_numel = numel == 0 ? 0 : ((numel + unit - 1) / unit) * unit;
  p.block = block;
  p.levels = levels;
  p.world = static_cast<int32_t>(world);
  p.rank = rank;
  p.w = w;
  p.s = s;
  p.gl = gl;
  int64_t stride = 1;
  for (int l = 0; l < levels; ++l) {
    p.group[l] = group[l];
    p.digit[l] = static_cast<int32_t>((rank / stride) % group[l]);
    stride *= group[l];
  }
  p.off[0] = 0;
  p.len[0] = p.padded_numel;
  for (int l = 1; l <= levels; ++l) {
    p.len[l] = p.len[l - 1] / group[l - 1];
    p.off[l] = p.off[l - 1] + p.digit[l - 1] * p.len[l];
  }
  *out = p;
  clear_error();
  return HZ_OK;
}

}  // namespace hz
