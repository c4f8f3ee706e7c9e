// hz_ctx and the engine helpers shared by engine.cpp (NCCL transport) and
// p2p.cpp (NVLink peer-memory transport).  Internal header.
#pragma once

#include <nccl.h>

#include <string>
#include <unordered_map>
#include <vector>

#include "hz_internal.h"

namespace hz {
struct VWorld;   // vworld.cpp
}

struct hz_ctx {
  int rank = 0, world = 1, levels = 0, device = 0;
  int group[HZ_MAX_LEVELS] = {0};
  int digit[HZ_MAX_LEVELS] = {0};
  ncclComm_t world_comm = nullptr;
  ncclComm_t lvl[HZ_MAX_LEVELS] = {nullptr};
  // merged qgZ hops over levels a..b (a < b), split lazily: hop_comm[a-1][b-1]
  ncclComm_t hop_comm[HZ_MAX_LEVELS][HZ_MAX_LEVELS] = {{nullptr}};
  bool nccl_dead = false;           // communicators aborted after an asynchronous error
  std::string nccl_err;
  struct Buf {
    void* p = nullptr;
    size_t cap = 0;
  };
  // NCCL transport workspace
  Buf ag_c, ag_s;                      // full-layer codes / scales (all-gather)
  Buf rs_a_c, rs_a_s, rs_b_c, rs_b_s;  // ping-pong send buffers (reduce-scatter)
  Buf rs_r_c, rs_r_s;                  // receive slots (reduce-scatter)
  Buf ar_a, ar_b, ar_g;                // allreduce + select: ping-pong fp32, gathered members

  // NVLink P2P transport (hz_enable_p2p / hz_init_virtual): one symmetric pool per rank.
  struct P2P {
    bool on = false;
    char* pool = nullptr;                       // local base
    size_t bytes = 0;
    size_t used = 0;                            // bump allocator (same on every rank)
    char* peer[hz::kMaxWorld] = {nullptr};      // every rank's pool base, mapped here
    unsigned long long phase = 0;               // last phase number issued (absolute)
    unsigned long long epoch_host = 0;          // value *epoch will hold once enqueued work ran
    unsigned long long capture_start = 0;       // phase at hz_p2p_capture_begin
    unsigned long long span = 0;                // phases of the last captured graph
    bool capturing = false;
    // prefetched quantize (hz_allgather_params_next): the next layer's primary was
    // quantized into pre_codes in phase pre_phase by the previous call's dual kernel,
    // with pre_bits / pre_dt / pre_len elements
    unsigned long long pre_phase = 0;
    const void* pre_codes = nullptr;
    const void* pre_primary = nullptr;
    int pre_bits = 0;
    hz_dtype pre_dt = HZ_BF16;
    int64_t pre_len = 0;
    struct Slot {
      size_t off = 0, cap = 0;
    };
    Slot ag_prim_c, ag_prim_s;                  // quantized primary when s != w
    // level-l qgZ send buffers; the last hop's input has two (alternating per reduce-scatter
    // call, rs_par): a call's deferred last hop still reads one while the next call writes
    // the other
    Slot rs_c[HZ_MAX_LEVELS + 1][2], rs_s[HZ_MAX_LEVELS + 1][2];
    int rs_par = 0;
    // deferred last qgZ hop of a hz_backward_step (p2p.cpp): run by the next call's
    // launch (the backward triple kernel) or flushed before any other phase
    struct PendRed {
      bool on = false;
      int g = 0;
      const uint8_t* c[hz::kMaxG] = {nullptr};
      const float* s[hz::kMaxG] = {nullptr};
      int64_t n = 0;
      int bits = 4;
      int block = 256;
      float* shard = nullptr;
      int acc = 0;
      int level = 0;
      unsigned long long ph = 0;   // its phase (wait ready >= ph from wr_mask)
      unsigned wr_mask = 0;
      int64_t remote = 0;
    } pend;
    Slot upd;                                   // updated weights of range_L (step tail)
    Slot ar_a, ar_b;                            // allreduce + select: ping-pong fp32 buffers
    // level-local synchronisation (host bookkeeping, p2p.cpp): the ranks this rank
    // reads from (its `done` signals go to them) and, per pool buffer, the ranks that
    // read this rank's copy of it (a writer of the buffer waits for their `done`)
    unsigned nbr = 0;
    std::unordered_map<size_t, unsigned> readers;
    // abort word in mapped page-locked host memory (device pointer for the kernels)
    unsigned* abort_host = nullptr;
    unsigned* abort_dev = nullptr;
    unsigned long long timeout_ns = 600ull * 1000000000ull;
    hz::VWorld* vw = nullptr;                   // virtual world (hz_init_virtual), else null
  } p2p;

  // Host-staged step executor (hz_step_host, executor.cpp): copy streams and events,
  // created on first use.
  struct Exec {
    cudaStream_t h2d = nullptr, d2h = nullptr;
    std::vector<cudaEvent_t> ev;        // 3 per tensor: primary in, grad in, shard ready
    cudaEvent_t kernels_done = nullptr; // the previous call's last kernel
    cudaEvent_t d2h_done = nullptr;
  } exec;
};

namespace hz {

// header of the symmetric pool: ready[8] u64 | done[8] u64 | arrival counter u32 |
// phase epoch u64
constexpr size_t kReadyOff = 0, kDoneOff = 64, kCounterOff = 128, kEpochOff = 192;
constexpr size_t kPoolHeader = 4096;

int tune_param(const char* name, int dflt);   // HZ_TUNE overrides (codec_util.cu)
hz_status cuda_fail(cudaError_t e, const char* what);
hz_status nccl_fail(ncclResult_t r, const char* what);
hz_status grow(hz_ctx::Buf& b, size_t need);
int64_t elem_bytes(hz_dtype dt);

// traced kernel launches (sync may be nullptr)
hz_status run_quantize(const void* x, hz_dtype dt, int64_t n, int bits, int block, uint8_t* c,
                       float* s, cudaStream_t st, int level, const SyncArgs* sync = nullptr);
hz_status run_dequantize(const uint8_t* c, const float* s, int64_t n, int bits, int block, void* y,
                         hz_dtype odt, cudaStream_t st, int level);
hz_status run_gather_dequantize(const Pieces& pc, int64_t n, int bits, int block, void* y,
                                hz_dtype odt, cudaStream_t st, int level, const SyncArgs* sync,
                                int64_t remote_bytes);
hz_status run_reduce(int g, const uint8_t* const* c, const float* const* s, int64_t n, int bits_in,
                     int block, int bits_out, uint8_t* oc, float* os, float* of, int acc,
                     cudaStream_t st, int level, const SyncArgs* sync = nullptr,
                     int64_t remote_bytes = 0);
hz_status run_gather_quantize_reduce(const Pieces& pc, int64_t n, void* y, const void* x, hz_dtype dt, int64_t nq,
                                     int qbits, uint8_t* c, float* s, int rg, const uint8_t* const* rc,
                                     const float* const* rs, int64_t rn, int rbits, float* shard, int acc, int level,
                                     cudaStream_t st, const SyncArgs& sync, int64_t remote_bytes);
hz_status run_gather_quantize(const Pieces& pc, int64_t n, int bits, void* y, hz_dtype odt, const void* x,
                              hz_dtype dt, int64_t nq, int qbits, uint8_t* c, float* s, cudaStream_t st,
                              const SyncArgs& sync, int64_t remote_bytes, float* qy = nullptr, int acc = 0);
hz_status copy_async(void* dst, const void* src, size_t bytes, cudaStream_t st);
hz_status run_sum(const Pieces& pc, int64_t n, float* out, cudaStream_t st, int level, const SyncArgs* sync,
                  int64_t remote);
hz_status p2p_allreduce_select(hz_ctx* ctx, const hz_partition_t* p, const float* in, int from_level, int to_level,
                               float* out, cudaStream_t st);

// P2P transport (p2p.cpp)
bool in_pool(const hz_ctx* ctx, const void* p, size_t bytes);
// partition made for this context (rank, world, levels, group sizes), valid block,
// padding and hop grouping (engine.cpp)
hz_status check_partition(const hz_ctx* ctx, const hz_partition_t* p);
// the next layer's quantize fused into this layer's forward gather (k_gather_quantize)
struct NextQ {
  const hz_partition_t* p;
  const void* primary;
  uint8_t* codes;
  float* scales;
};
// the previous layer's backward gather fused into this layer's level-`from` quantize
struct PrevG {
  const hz_partition_t* p;
  uint8_t* sec_codes;
  float* sec_scales;
  int bits;
  void* full_out;
  hz_dtype out_dt;
};
bool p2p_next_fusable(const hz_ctx* ctx, const hz_partition_t* p, int bits, hz_dtype out_dt, const NextQ& nx);
hz_status p2p_allgather(hz_ctx* ctx, const hz_partition_t* p, int backward, const void* primary,
                        hz_dtype dt, int bits, uint8_t* sec_codes, float* sec_scales, void* full_out,
                        hz_dtype out_dt, cudaStream_t st, const NextQ* next);
bool p2p_prev_fusable(const hz_ctx* ctx, const hz_partition_t* p, int from_level, const PrevG& pg);
hz_status p2p_reduce_scatter(hz_ctx* ctx, const hz_partition_t* p, const void* grad, hz_dtype dt,
                             int from_level, int to_level, const int* bits_per_level, float* shard,
                             int accumulate, cudaStream_t st, const PrevG* prev = nullptr);
void p2p_release(hz_ctx* ctx);
hz_status p2p_alloc_abort(hz_ctx* ctx);
hz_status p2p_check(const hz_ctx* ctx);        // HZ_ERR_ABORTED once the context is aborted
hz_status check_async(const hz_ctx* ctx);      // asynchronous NCCL errors of every communicator (engine.cpp)
// virtual world (vworld.cpp): host-side ordering of one synchronised launch
hz_status vw_wait(hz_ctx* ctx, const SyncArgs& s, cudaStream_t st);
hz_status vw_signal(hz_ctx* ctx, const SyncArgs& s, cudaStream_t st);
void vw_abort(hz_ctx* ctx);
void vw_release(hz_ctx* ctx);
void exec_release(hz_ctx* ctx);   // executor.cpp
hz_status p2p_adamw_gather(hz_ctx* ctx, const hz_partition_t* p, const float* g, float* th, float* m, float* v,
                           const AdamW& hp, void* primary, hz_dtype dt, cudaStream_t st);
hz_status run_adamw(const float* g, float* th, float* m, float* v, void* out, hz_dtype dt, int64_t n,
                    const AdamW& hp, cudaStream_t st, const SyncArgs* sync);

}  // namespace hz
