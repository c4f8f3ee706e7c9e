// Communication plans (host only): the exact sequence of per-level NCCL
// operations one rank issues for hz_allgather_params / hz_reduce_scatter_grads.
// The engine (engine.cpp) issues its NCCL calls from these plans, and the CPU
// gloo tests execute the same plans with gloo transport to check that every
// send has a matching receive with the same offsets and sizes on the peer.
//
//   all-gather (O7/O8, Table VII): for l = top..1 with g_l > 1:
//       ALLGATHER(level l, piece = range_l (len_l elems), into range_{l-1})
//     top = w (forward) or s (backward).
//   reduce-scatter (O9, Table VIII): for every hop a..b of p's grouping
//     inside from..to (one hop per level by default), for every member j != me of
//     the hop group in ascending merged digit (= ascending rank):
//       SENDRECV(hop a..b, peer j, send member j's chunk of range_{a-1}, receive range_b)
#include <string>
#include <vector>

#include "hz_internal.h"

namespace hz {

hz_status plan_allgather(const hz_partition_t* p, int backward, int bits, std::vector<hz_comm_step>* out) {
  if (!p) return fail(HZ_ERR_INVALID, "p: NULL");
  if (!bits_ok(bits)) return fail(HZ_ERR_INVALID, "bits: must be 4 or 8");
  out->clear();
  const int top = backward ? p->s : p->w;
  for (int l = top; l >= 1; --l) {
    const int g = p->group[l - 1];
    if (g <= 1) continue;
    hz_comm_step st{};
    st.op = HZ_PLAN_ALLGATHER;
    st.level = l;
    st.level_last = l;
    st.group = g;
    st.peer = -1;
    st.peer_rank = -1;
    st.bits = bits;
    st.elems = p->len[l];
    st.send_off = p->off[l];
    st.recv_off = p->off[l - 1];
    st.code_bytes = code_bytes(p->len[l], bits);
    st.scale_bytes = p->len[l] / p->block * 4;
    out->push_back(st);
  }
  return HZ_OK;
}

hz_status plan_reduce_scatter(const hz_partition_t* p, int from_level, int to_level,
                              const int* bits_per_level, std::vector<hz_comm_step>* out) {
  if (!p) return fail(HZ_ERR_INVALID, "p: NULL");
  const int L = p->levels;
  if (from_level < 1 || from_level > L) return fail(HZ_ERR_INVALID, "from_level: must be in [1, levels]");
  if (to_level < from_level || to_level > L) return fail(HZ_ERR_INVALID, "to_level: must be in [from_level, levels]");
  if (!bits_per_level) return fail(HZ_ERR_INVALID, "bits_per_level: NULL");
  out->clear();
  std::vector<Hop> hops;
  hz_status rc = hops_of(p, from_level, to_level, &hops);
  if (rc != HZ_OK) return rc;
  std::vector<int> ranks;
  std::vector<int64_t> rel;
  for (const Hop& h : hops) {
    const int bits = bits_per_level[h.a - 1];
    if (!bits_ok(bits)) return fail(HZ_ERR_INVALID, "bits_per_level[" + std::to_string(h.a - 1) + "]: must be 4 or 8");
    int me = 0;
    hop_members(p, h.a, h.b, &ranks, &rel, &me);
    const int G = static_cast<int>(ranks.size());
    for (int j = 0; j < G; ++j) {
      if (j == me) continue;
      hz_comm_step st{};
      st.op = HZ_PLAN_SENDRECV;
      st.level = h.a;
      st.level_last = h.b;
      st.group = G;
      st.peer = j;
      st.peer_rank = ranks[j];
      st.bits = bits;
      st.elems = p->len[h.b];
      st.send_off = p->off[h.a - 1] + rel[j];
      st.recv_off = p->off[h.b];
      st.code_bytes = code_bytes(p->len[h.b], bits);
      st.scale_bytes = p->len[h.b] / p->block * 4;
      out->push_back(st);
    }
  }
  return HZ_OK;
}

namespace {
hz_status copy_out(const std::vector<hz_comm_step>& v, hz_comm_step* out, int max, int* n_out) {
  if (!n_out) return fail(HZ_ERR_INVALID, "n_out: NULL");
  if (max > 0 && !out) return fail(HZ_ERR_INVALID, "out: NULL");
  const int n = static_cast<int>(v.size());
  for (int i = 0; i < n && i < max; ++i) out[i] = v[i];
  *n_out = n;
  clear_error();
  return HZ_OK;
}
}  // namespace

}  // namespace hz

extern "C" {

hz_status hz_plan_allgather(const hz_partition_t* p, int backward, int bits, hz_comm_step* out, int max,
                            int* n_out) {
  std::vector<hz_comm_step> v;
  hz_status rc = hz::plan_allgather(p, backward, bits, &v);
  if (rc != HZ_OK) return rc;
  return hz::copy_out(v, out, max, n_out);
}

hz_status hz_plan_reduce_scatter(const hz_partition_t* p, int from_level, int to_level,
                                 const int* bits_per_level, hz_comm_step* out, int max, int* n_out) {
  std::vector<hz_comm_step> v;
  hz_status rc = hz::plan_reduce_scatter(p, from_level, to_level, bits_per_level, &v);
  if (rc != HZ_OK) return rc;
  return hz::copy_out(v, out, max, n_out);
}

}  // extern "C"
