// C-ABI surface of libhz.so: error reporting, argument validation and the
// standalone codec entry points (hz_quantize / hz_dequantize / hz_reduce_chunks).
// The collectives live in engine.cpp, tracing in trace.cpp.
#include <cstdint>
#include <string>

#include "hz_internal.h"

namespace hz {
namespace {
thread_local std::string t_err;
}

hz_status fail(hz_status st, const std::string& msg) {
  t_err = msg;
  return st;
}

void clear_error() { t_err.clear(); }

bool block_ok(int block) { return block >= 32 && block <= 2048 && (block & (block - 1)) == 0; }

bool bits_ok(int bits) { return bits == 4 || bits == 8; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int64_t code_bytes(int64_t n, int bits) { return n * bits / 8; }

namespace {
hz_status launch_status(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(HZ_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  clear_error();
  return HZ_OK;
}

hz_status check_codec(int64_t n, int bits, int block) {
  if (n < 0) return fail(HZ_ERR_INVALID, "n: negative");
  if (!bits_ok(bits)) return fail(HZ_ERR_INVALID, "bits: must be 4 or 8");
  if (!block_ok(block)) return fail(HZ_ERR_INVALID, "block: must be a power of two in [32, 2048]");
  if (n % block) return fail(HZ_ERR_INVALID, "n: must be a multiple of block");
  return HZ_OK;
}

const char* const kSymbols[] = {
    "hz_version",          "hz_last_error",          "hz_num_symbols",
    "hz_symbol_name",      "hz_partition_ex",        "hz_quantize",
    "hz_dequantize",       "hz_reduce_chunks",       "hz_get_uid",
    "hz_init",             "hz_finalize",            "hz_partition",
    "hz_allgather_params", "hz_reduce_scatter_grads", "hz_flat_allgather",
    "hz_flat_reduce_scatter", "hz_trace_begin",      "hz_trace_end",
    "hz_trace_read",       "hz_plan_allgather",      "hz_plan_reduce_scatter",
    "hz_enable_p2p",       "hz_p2p_enabled",         "hz_sym_alloc",
    "hz_p2p_capture_begin", "hz_p2p_capture_end",    "hz_p2p_replayed",
    "hz_adamw_step",       "hz_set_sm_budget",     "hz_allreduce_select", "hz_step_host", "hz_allgather_params_next", "hz_backward_step",
    "hz_partition_set_hops", "hz_init_virtual",    "hz_init_virtual_ex",    "hz_set_wait_timeout",
    "hz_abort",            "hz_check",             "hz_adamw_params",
    "hz_nvlink_probe",     "hz_flush",
};
}  // namespace
}  // namespace hz

extern "C" {

const char* hz_version(void) { return "hz 0.1 sm_100a"; }

const char* hz_last_error(void) { return hz::t_err.c_str(); }

int hz_num_symbols(void) { return static_cast<int>(sizeof(hz::kSymbols) / sizeof(hz::kSymbols[0])); }

const char* hz_symbol_name(int i) {
  if (i < 0 || i >= hz_num_symbols()) return nullptr;
  return hz::kSymbols[i];
}

hz_status hz_partition_ex(int rank, int levels, const int* group, int64_t numel, int block, int w,
                          int s, int gl, hz_partition_t* out) {
  return hz::partition(rank, levels, group, numel, block, w, s, gl, out);
}

hz_status hz_quantize(const void* x, hz_dtype dt, int64_t n, int bits, int block, uint8_t* codes,
                      float* scales, void* stream) {
  using namespace hz;
  hz_status rc = check_codec(n, bits, block);
  if (rc != HZ_OK) return rc;
  if (dt != HZ_F32 && dt != HZ_BF16 && dt != HZ_F16) return fail(HZ_ERR_INVALID, "dt: unknown dtype");
  if (n == 0) {
    clear_error();
    return HZ_OK;
  }
  if (!x || !aligned16(x)) return fail(HZ_ERR_INVALID, "x: NULL or not 16-byte aligned");
  if (!codes || !aligned16(codes)) return fail(HZ_ERR_INVALID, "codes: NULL or not 16-byte aligned");
  if (!scales || !aligned16(scales)) return fail(HZ_ERR_INVALID, "scales: NULL or not 16-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  TraceScope t(st, "quantize", 0, bits, n, n * (dt == HZ_F32 ? 4 : 2) + code_bytes(n, bits) + n / block * 4);
  SyncArgs sy{};
  sy.stamps = t.stamps;
  cudaError_t e = launch_quantize(x, dt, n, bits, block, codes, scales, st, t.stamps ? &sy : nullptr);
  t.end();
  return launch_status(e, "quantize kernel launch");
}

hz_status hz_dequantize(const uint8_t* codes, const float* scales, int64_t n, int bits, int block,
                        void* y, hz_dtype out_dt, void* stream) {
  using namespace hz;
  hz_status rc = check_codec(n, bits, block);
  if (rc != HZ_OK) return rc;
  if (out_dt != HZ_F32 && out_dt != HZ_BF16 && out_dt != HZ_F16)
    return fail(HZ_ERR_INVALID, "out_dt: unknown dtype");
  if (n == 0) {
    clear_error();
    return HZ_OK;
  }
  if (!codes || !aligned16(codes)) return fail(HZ_ERR_INVALID, "codes: NULL or not 16-byte aligned");
  if (!scales || !aligned16(scales)) return fail(HZ_ERR_INVALID, "scales: NULL or not 16-byte aligned");
  if (!y || !aligned16(y)) return fail(HZ_ERR_INVALID, "y: NULL or not 16-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  TraceScope t(st, "dequantize", 0, bits, n, code_bytes(n, bits) + n / block * 4 + n * (out_dt == HZ_F32 ? 4 : 2));
  Pieces pc{};
  pc.c[0] = codes;
  pc.s[0] = scales;
  pc.n = 1;
  pc.len = n;
  SyncArgs sy{};
  sy.stamps = t.stamps;
  cudaError_t e = launch_gather_dequantize(pc, n, bits, block, y, out_dt, st, t.stamps ? &sy : nullptr);
  t.end();
  return launch_status(e, "dequantize kernel launch");
}

hz_status hz_reduce_chunks(int g, const uint8_t* const* codes, const float* const* scales,
                           int64_t n, int bits_in, int block, int bits_out, uint8_t* out_codes,
                           float* out_scales, float* out_f32, int accumulate, void* stream) {
  using namespace hz;
  if (g < 1 || g > kMaxG) return fail(HZ_ERR_INVALID, "g: must be in [1, 16]");
  hz_status rc = check_codec(n, bits_in, block);
  if (rc != HZ_OK) return rc;
  if (bits_out != 0 && !bits_ok(bits_out)) return fail(HZ_ERR_INVALID, "bits_out: must be 0, 4 or 8");
  if (n == 0) {
    clear_error();
    return HZ_OK;
  }
  if (!codes || !scales) return fail(HZ_ERR_INVALID, "codes/scales: NULL pointer array");
  for (int p = 0; p < g; ++p) {
    if (!codes[p] || !aligned16(codes[p]))
      return fail(HZ_ERR_INVALID, "codes[" + std::to_string(p) + "]: NULL or not 16-byte aligned");
    if (!scales[p] || !aligned16(scales[p]))
      return fail(HZ_ERR_INVALID, "scales[" + std::to_string(p) + "]: NULL or not 16-byte aligned");
  }
  if (bits_out) {
    if (!out_codes || !aligned16(out_codes)) return fail(HZ_ERR_INVALID, "out_codes: NULL or not 16-byte aligned");
    if (!out_scales || !aligned16(out_scales)) return fail(HZ_ERR_INVALID, "out_scales: NULL or not 16-byte aligned");
  } else if (!out_f32 || !aligned16(out_f32)) {
    return fail(HZ_ERR_INVALID, "out_f32: NULL or not 16-byte aligned");
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t in_bytes = g * (code_bytes(n, bits_in) + n / block * 4);
  const int64_t out_bytes = bits_out ? code_bytes(n, bits_out) + n / block * 4 : n * 4 * (accumulate ? 2 : 1);
  TraceScope t(st, bits_out ? "reduce_requant" : "reduce", 0, bits_in, n, in_bytes + out_bytes);
  SyncArgs sy{};
  sy.stamps = t.stamps;
  cudaError_t e = launch_reduce(g, codes, scales, n, bits_in, block, bits_out, out_codes, out_scales,
                                out_f32, accumulate, st, t.stamps ? &sy : nullptr);
  t.end();
  return launch_status(e, "reduce kernel launch");
}

}  // extern "C"
