// Internal declarations shared by the libhz.so translation units (not installed).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/hz.h"

namespace hz {

// thread-local error message (abi.cpp)
hz_status fail(hz_status st, const std::string& msg);
void clear_error();

// --------------------------------------------------------------- validation
bool block_ok(int block);          // power of two in [32, 2048]
bool bits_ok(int bits);            // 4 or 8
bool aligned16(const void* p);
int64_t code_bytes(int64_t n, int bits);   // n * bits / 8

// ------------------------------------------------------------- P2P phase sync
// (see codec.cuh for the protocol).  A zero-initialised SyncArgs means "no sync".
constexpr int kMaxWorld = 8;
constexpr unsigned kWaitReady = 1u, kWaitDone = 2u, kSigReady = 4u, kSigDone = 8u;
struct SyncArgs {
  unsigned long long* ready_local;
  unsigned long long* done_local;
  unsigned long long* ready_remote[kMaxWorld];
  unsigned long long* done_remote[kMaxWorld];
  unsigned int* counter;
  int world;
  // phase thresholds relative to *epoch (the device-side phase offset advanced by
  // every replay of a captured CUDA graph); `en` says which of them are active
  unsigned long long wait_ready, wait_done, sig_ready, sig_done;
  const unsigned long long* epoch;
  unsigned en;   // kWaitReady | kWaitDone | kSigReady | kSigDone
  unsigned long long* stamps;   // optional [8]: entry, after wait, last-CTA arrival, flags sent (ns), counter
  int mode;                     // publication fence variant (HZ_TUNE p2p_sig; 0 = fence.sc.sys)
  int sysfence;                 // per-CTA fence at system scope (kernels that store into peer memory)
};

// Pieces of a gathered layer for the fused gather+dequantize kernel: piece j
// covers elements [j*len, (j+1)*len) and its codes / scales are read from
// (possibly peer-mapped) c[j] / s[j].  n == 1 with c[0], s[0] is a plain
// dequantize.  Optionally the codes of [sec_lo, sec_hi) are also copied into
// sec_c / sec_s (hpZ secondary kept from a flattened gather).
struct Pieces {
  const uint8_t* c[kMaxWorld];
  const float* s[kMaxWorld];
  int n;
  int64_t len;
  uint8_t* sec_c;
  float* sec_s;
  int64_t sec_lo, sec_hi;
  // hybrid push/pull: elements [0, split) of piece j come from cr[j] / sr[j] (local
  // receive buffer) when cr[j] is set
  const uint8_t* cr[kMaxWorld];
  const float* sr[kMaxWorld];
  int64_t split;
};

// ----------------------------------------------------------------- kernels
// All launchers validate nothing (the ABI layer does) and return cudaGetLastError().
// `sync` may be nullptr (no cross-GPU phase synchronisation).
cudaError_t launch_quantize(const void* x, hz_dtype dt, int64_t n, int bits, int block,
                            uint8_t* codes, float* scales, cudaStream_t st,
                            const SyncArgs* sync = nullptr);
// Fused quantize + dequantize (a level whose exchange group has one member): codes
// and scales as launch_quantize, plus y = out_dt(fl(code*scale)) (fp32: += when acc).
// block must be 256 (roundtrip_supported).
bool roundtrip_supported(int block);
cudaError_t launch_quantize_roundtrip(const void* x, hz_dtype dt, int64_t n, int bits, int block,
                                      uint8_t* codes, float* scales, void* y, hz_dtype out_dt, int acc,
                                      cudaStream_t st, const SyncArgs* sync);
// Dual kernel (k_quantize.cu): gather+dequantize of pc (n_gather elements, 8-bit codes,
// bf16 out, B = 256) and quantize of x (n_q elements, qbits) in one launch.
bool gather_quantize_supported(int block, int gather_bits, hz_dtype out_dt);
// qy != nullptr: the quantize job is the fp32 round trip of a one-member level (x_hat
// into qy, += when acc; codes / scales not stored).
cudaError_t launch_gather_quantize(const Pieces& pc, int64_t n_gather, void* y, const void* x, hz_dtype dt,
                                   int64_t n_q, int qbits, uint8_t* codes, float* scales, float* qy, int acc,
                                   cudaStream_t st, const SyncArgs& sy);
cudaError_t launch_dequantize(const uint8_t* codes, const float* scales, int64_t n, int bits,
                              int block, void* y, hz_dtype out_dt, cudaStream_t st);
cudaError_t launch_gather_dequantize(const Pieces& pc, int64_t n, int bits, int block, void* y,
                                     hz_dtype out_dt, cudaStream_t st, const SyncArgs* sync);
constexpr int kMaxG = 16;

// Push destinations of the P2P push kernels (quantize / requantize that store their
// codes straight into the consumers' receive buffers over NVLink).  The codes and
// scales of element e go, besides the local buffers (if any), to every c[j] + e
// (mirror), or only to segment j = e / seg at c[j] + (e - j*seg) (scatter).
struct PushDst {
  uint8_t* c[kMaxG];
  float* s[kMaxG];
  int64_t seg;      // scatter segment in elements (a multiple of the block)
  int n;
  int scatter;
  int64_t lim;      // > 0: only elements whose offset (within the segment) is < lim
};
// Push variants (P2P transport, block 256): codes / scales also (or only, when
// codes == nullptr) stored to `dst` (peer receive buffers); y (optional) = the own
// round trip x_hat.  The per-CTA release fences at system scope.
cudaError_t launch_quantize_push(const void* x, hz_dtype dt, int64_t n, int bits, uint8_t* codes, float* scales,
                                 void* y, hz_dtype out_dt, const PushDst& dst, cudaStream_t st,
                                 const SyncArgs* sync);
bool push_reduce_supported(int g, int block);
cudaError_t launch_reduce_push(int g, const uint8_t* const* codes, const float* const* scales, int64_t n,
                               int bits_in, int bits_out, const PushDst& dst, cudaStream_t st,
                               const SyncArgs* sync);

cudaError_t launch_epoch_advance(unsigned long long* epoch, unsigned long long span, cudaStream_t st);
cudaError_t launch_reduce(int g, const uint8_t* const* codes, const float* const* scales,
                          int64_t n, int bits_in, int block, int bits_out, uint8_t* out_codes,
                          float* out_scales, float* out_f32, int accumulate, cudaStream_t st,
                          const SyncArgs* sync = nullptr);

// Step tail (k_optim.cu): AdamW on the optimizer shard and the bf16/fp16/fp32
// gather copy of the post-update all-gather.  Same layout as hz_adamw_t.
struct AdamW {
  float b1, omb1, b2, omb2, lr_wd, sqrt_bc2, eps, step;
};
cudaError_t launch_adamw(const float* g, float* th, float* m, float* v, void* out, hz_dtype out_dt, int64_t n,
                         const AdamW& hp, cudaStream_t st, const SyncArgs* sync);
cudaError_t launch_gather_copy(const Pieces& pc, void* out, cudaStream_t st, const SyncArgs* sync);
// out[i] = ((c[0][i] + c[1][i]) + ...) + c[n-1][i] over fp32 pieces (Pieces::c as
// float arrays of n elements, n % 4 == 0; the pieces may be peer-mapped)
cudaError_t launch_sum_f32(const Pieces& pc, int64_t n, float* out, cudaStream_t st, const SyncArgs* sync);

// Fused codec + NVLink collective kernels (k_fused.cu, B = 256 only).
constexpr int kMaxChunks = 4096;   // per-chunk flags per member in the P2P pool header
struct FusedAGArgs {
  const void* x;
  hz_dtype dt;
  int bits;
  uint8_t* qc;
  float* qs;
  const uint8_t* pc[kMaxWorld];
  const float* ps[kMaxWorld];
  int D, me;
  int64_t plen, C;
  int nch;
  unsigned long long* flags;
  unsigned long long* flags_remote[kMaxWorld];
  unsigned long long* work;
  unsigned int* cnt;      // per-chunk producer arrival counters (local, zero between launches)
  unsigned long long* dbg;   // optional per-chunk timeline (HZ_TUNE pdbg)
  void* y;
  hz_dtype out_dt;
  unsigned long long phase;
  const unsigned long long* epoch;
};
struct FusedRSArgs {
  const void* x;
  hz_dtype dt;
  int bits_in, bits_out, acc;
  uint8_t* qc;
  float* qs;
  const uint8_t* mc[kMaxG];
  const float* ms[kMaxG];
  int g, d;
  int64_t cl, C;
  int ncl;
  unsigned long long* flags;
  unsigned long long* flags_remote[kMaxG];
  unsigned long long* work;
  unsigned int* cnt;
  float* of;
  uint8_t* oc;
  float* os;
  unsigned long long phase;
  const unsigned long long* epoch;
};
bool fused_rs_supported(int g);
cudaError_t launch_ag_fused(const FusedAGArgs& a, cudaStream_t st, const SyncArgs& sy);
cudaError_t launch_rs_fused(const FusedRSArgs& a, cudaStream_t st, const SyncArgs& sy);

// ------------------------------------------------------------------ tracing
struct TraceScope {
  // Records a start event on construction and an end event + record on end().
  // bytes = algorithmic bytes of this GPU's HBM; remote = bytes read from peers over NVLink
  TraceScope(cudaStream_t st, const char* kind, int level, int bits, int64_t elems,
             int64_t bytes, int64_t remote = 0);
  void end();
  ~TraceScope();
  bool active;
  int slot;
  cudaStream_t stream;
  unsigned long long* stamps;   // device [3] for this launch when tracing, else nullptr
};

// ----------------------------------------------------------------- partition
hz_status partition(int rank, int levels, const int* group, int64_t numel, int block, int w,
                    int s, int gl, hz_partition_t* out);

// -------------------------------------------------------------------- plans
hz_status plan_allgather(const hz_partition_t* p, int backward, int bits, std::vector<hz_comm_step>* out);
hz_status plan_reduce_scatter(const hz_partition_t* p, int from_level, int to_level,
                              const int* bits_per_level, std::vector<hz_comm_step>* out);

}  // namespace hz
