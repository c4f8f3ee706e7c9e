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

// ------------------------------------------------- shared-memory carveout
// Preferred shared-memory carveout (percent, -1 = driver default) that launch_k_smem
// (codec.cuh) attaches to every libhz launch of this host thread, set per API call by
// CarveScope.  A world-1 context uses 100 (HZ_TUNE carve1): with every kernel of its
// sequence at one carveout, the SMs need no shared-memory reconfiguration between the
// dequantize and round-trip launches (N = 1 step 3.233 vs 3.278 ms, round trip 49.1 vs
// 49.9 us; profiles/tma_r02.md, carveout addendum).  World > 1 keeps the driver default
// (HZ_TUNE carve): the P2P kernels read through L1 and measured slower at 100 (N = 2 step
// 4.32 vs 3.93 ms).
int launch_carve();
struct CarveScope {
  int prev;
  explicit CarveScope(int world);
  ~CarveScope();
};

// --------------------------------------------------------------- validation
bool block_ok(int block);          // power of two in [32, 2048]
bool bits_ok(int bits);            // 4 or 8
bool aligned16(const void* p);
int64_t code_bytes(int64_t n, int bits);   // n * bits / 8

// ------------------------------------------------------------- P2P phase sync
// (see codec.cuh for the protocol).  A zero-initialised SyncArgs means "no sync".
constexpr int kMaxWorld = 8;
struct SyncArgs {
  unsigned long long* ready_local;               // this rank's flags: ready[q] / done[q] =
  unsigned long long* done_local;                // the last phase rank q signalled to this rank
  unsigned long long* ready_remote[kMaxWorld];   // &ready[me] / &done[me] in rank q's pool
  unsigned long long* done_remote[kMaxWorld];
  unsigned int* counter;                         // last-CTA arrival counter (pool header)
  const unsigned long long* epoch;
  unsigned int* abort;             // mapped host word: nonzero = the context is aborted
  unsigned long long timeout_ns;   // a wait longer than this aborts (sets *abort = 1)
  // wait until ready[q] >= wait_ready for q in wr_mask and done[q] >= wait_done for q
  // in wd_mask; signal sig_ready to the ranks of sr_mask and sig_done to sd_mask.
  // Phase numbers are relative to *epoch (the device-side offset advanced by every
  // replay of a captured CUDA graph).
  unsigned long long wait_ready, wait_done, sig_ready, sig_done;
  unsigned wr_mask, wd_mask, sr_mask, sd_mask;
  unsigned long long* stamps;      // optional [8]: entry, after wait, last-CTA arrival, flags sent (ns), counter
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
// The TMA tile engine (k_tiles.cu): the same operations as the launchers above with
// every byte moved by bulk copy.  Each returns cudaErrorNotSupported (nothing launched)
// when the shape does not qualify: block != 256, a length not a multiple of 1024, a
// buffer not 16-byte aligned, an accumulating round trip, HZ_TUNE tma=0.
bool tiles_on();
cudaError_t tiles_quantize(const void* x, hz_dtype dt, int64_t n, int bits, int block, uint8_t* codes, float* scales,
                           void* y, hz_dtype out_dt, int acc, cudaStream_t st, const SyncArgs& sy);
cudaError_t tiles_gather(const Pieces& pc, int bits, int block, void* y, hz_dtype out_dt, cudaStream_t st,
                         const SyncArgs& sy);
cudaError_t tiles_dual(const Pieces& pc, void* y, const void* x, hz_dtype dt, int64_t nq, int qbits, uint8_t* codes,
                       float* scales, float* qy, int acc, cudaStream_t st, const SyncArgs& sy);
cudaError_t tiles_reduce(int g, const uint8_t* const* c, const float* const* s, int64_t n, int bits_in, int block,
                         int bits_out, uint8_t* oc, float* os, float* of, int acc, cudaStream_t st,
                         const SyncArgs& sy);
// Backward triple kernel (k_reduce.cu): the dual kernel's gather (8-bit, bf16 out) and
// quantize plus the fp32 level reduce of g (2 or 4) coded inputs into `shard` (+= when
// acc), one launch.  B = 256.
bool gather_quantize_reduce_supported(int gather_bits, hz_dtype out_dt, int g, int red_bits);
cudaError_t launch_gather_quantize_reduce(const Pieces& pc, int64_t n_gather, void* y, const void* x, hz_dtype dt,
                                          int64_t n_q, int qbits, uint8_t* codes, float* scales, int g,
                                          const uint8_t* const* rc, const float* const* rs, int64_t rn, int rbits,
                                          float* shard, int acc, cudaStream_t st, const SyncArgs& sy);
cudaError_t launch_dequantize(const uint8_t* codes, const float* scales, int64_t n, int bits,
                              int block, void* y, hz_dtype out_dt, cudaStream_t st);
cudaError_t launch_gather_dequantize(const Pieces& pc, int64_t n, int bits, int block, void* y,
                                     hz_dtype out_dt, cudaStream_t st, const SyncArgs* sync);
constexpr int kMaxG = 16;

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
// NVLink probe (hz_nvlink_probe): read `bytes` of (peer) memory at src, XOR into sink[grid]
cudaError_t launch_peer_read(const void* src, int64_t bytes, unsigned* sink, cudaStream_t st);
// out[i] = ((c[0][i] + c[1][i]) + ...) + c[n-1][i] over fp32 pieces (Pieces::c as
// float arrays of n elements, n % 4 == 0; the pieces may be peer-mapped)
cudaError_t launch_sum_f32(const Pieces& pc, int64_t n, float* out, cudaStream_t st, const SyncArgs* sync);

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

// qgZ hops (partition.cpp): levels a..b exchanged in one all-to-all
struct Hop {
  int a, b;
};
hz_status hops_of(const hz_partition_t* p, int from_level, int to_level, std::vector<Hop>* out);
void hop_members(const hz_partition_t* p, int a, int b, std::vector<int>* ranks, std::vector<int64_t>* rel,
                 int* me);

// -------------------------------------------------------------------- plans
hz_status plan_allgather(const hz_partition_t* p, int backward, int bits, std::vector<hz_comm_step>* out);
hz_status plan_reduce_scatter(const hz_partition_t* p, int from_level, int to_level,
                              const int* bits_per_level, std::vector<hz_comm_step>* out);

}  // namespace hz
