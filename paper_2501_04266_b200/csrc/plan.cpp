// Communication plans (host only): the exact sequence of per-level NCCL
// operations one rank issues for hz_allgather_params / hz_reduce_scatter_grads.
// The engine (engine.cpp) issues its NCCL calls from these plans, and the CPU
// gloo tests execute the same plans with gloo transport to check that every
// send has a matching receive with the same offsets and sizes on the peer.
//
//   all-gather (O7/O8, Table VII): for l = top..1 with g_l > 1:
//       ALLGATHER(level l, piece = range_l (len_l elems), into range_{l-1})
//     top = w (forward) or s (backward).
//   reduce-scatter (O9, Table VIII): for l = from..to with g_l > 1, for
//     every peer digit j != d_l in ascending order:
//       SENDRECV(level l, peer j, send chunk j of range_{l-1}, receive range_l)
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
  int64_t stride[HZ_MAX_LEVELS];
  int64_t s = 1;
  for (int l = 0; l < L; ++l) {
    stride[l] = s;
    s *= p->group[l];
  }
  for (int l = from_level; l <= to_level; ++l) {
    const int bits = bits_per_level[l - 1];
    if (!bits_ok(bits)) return fail(HZ_ERR_INVALID, "bits_per_level[" + std::to_string(l - 1) + "]: must be 4 or 8");
    const int g = p->group[l - 1];
    const int d = p->digit[l - 1];
    for (int j = 0; j < g; ++j) {
      if (j == d) continue;
      hz_comm_step st{};
      st.op = HZ_PLAN_SENDRECV;
      st.level = l;
      st.group = g;
      st.peer = j;
      st.peer_rank = static_cast<int32_t>(p->rank + (static_cast<int64_t>(j) - d) * stride[l - 1]);
      st.bits = bits;
      st.elems = p->len[l];
      st.send_off = p->off[l - 1] + j * p->len[l];
      st.recv_off = p->off[l];
      st.code_bytes = code_bytes(p->len[l], bits);
      st.scale_bytes = p->len[l] / p->block * 4;
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
