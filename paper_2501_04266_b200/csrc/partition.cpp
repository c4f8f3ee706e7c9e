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
#include <vector>

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

// qgZ hop grouping (R15): the hops of p inside levels from..to.
hz_status hops_of(const hz_partition_t* p, int from_level, int to_level, std::vector<Hop>* out) {
  out->clear();
  if (p->nhops <= 0) {
    for (int l = from_level; l <= to_level; ++l) out->push_back(Hop{l, l});
    return HZ_OK;
  }
  int a = 1;
  for (int k = 0; k < p->nhops; ++k) {
    const int b = p->hop_last[k];
    if (a >= from_level && b <= to_level) {
      out->push_back(Hop{a, b});
    } else if ((a < from_level && b >= from_level) || (a <= to_level && b > to_level)) {
      return fail(HZ_ERR_INVALID, "from_level/to_level: must fall on hop boundaries of p (hop levels " +
                                      std::to_string(a) + ".." + std::to_string(b) + ")");
    }
    a = b + 1;
  }
  return HZ_OK;
}

// Members of p's rank in the hop over levels a..b, ascending rank (= ascending merged
// digit j = sum_{l=a..b} d_l * prod_{k=a}^{l-1} g_k), with rel = off_b(member) -
// off_{a-1}: where the member's chunk lies in range_{a-1}.
void hop_members(const hz_partition_t* p, int a, int b, std::vector<int>* ranks, std::vector<int64_t>* rel,
                 int* me) {
  int64_t stride[HZ_MAX_LEVELS];
  int64_t st = 1;
  for (int l = 0; l < p->levels; ++l) {
    stride[l] = st;
    st *= p->group[l];
  }
  int64_t base = p->rank;
  int64_t G = 1;
  for (int l = a; l <= b; ++l) {
    base -= p->digit[l - 1] * stride[l - 1];
    G *= p->group[l - 1];
  }
  ranks->clear();
  rel->clear();
  for (int64_t j = 0; j < G; ++j) {
    int64_t rem = j, r = base, off = 0;
    for (int l = a; l <= b; ++l) {
      const int64_t d = rem % p->group[l - 1];
      rem /= p->group[l - 1];
      r += d * stride[l - 1];
      off += d * p->len[l];
    }
    if (r == p->rank && me) *me = static_cast<int>(j);
    ranks->push_back(static_cast<int>(r));
    rel->push_back(off);
  }
}

}  // namespace hz

extern "C" hz_status hz_partition_set_hops(hz_partition_t* p, int nhops, const int* hop_last) {
  using namespace hz;
  if (!p) return fail(HZ_ERR_INVALID, "p: NULL");
  if (nhops == 0) {
    p->nhops = 0;
    for (int k = 0; k < HZ_MAX_LEVELS; ++k) p->hop_last[k] = 0;
    clear_error();
    return HZ_OK;
  }
  if (nhops < 0 || nhops > p->levels) return fail(HZ_ERR_INVALID, "nhops: must be in [0, levels]");
  if (!hop_last) return fail(HZ_ERR_INVALID, "hop_last: NULL");
  int prev = 0;
  for (int k = 0; k < nhops; ++k) {
    if (hop_last[k] <= prev || hop_last[k] > p->levels)
      return fail(HZ_ERR_INVALID, "hop_last[" + std::to_string(k) + "]: must be strictly ascending in [1, levels]");
    prev = hop_last[k];
  }
  if (prev != p->levels) return fail(HZ_ERR_INVALID, "hop_last: the last hop must end at level L");
  p->nhops = nhops;
  for (int k = 0; k < HZ_MAX_LEVELS; ++k) p->hop_last[k] = k < nhops ? hop_last[k] : 0;
  clear_error();
  return HZ_OK;
}
