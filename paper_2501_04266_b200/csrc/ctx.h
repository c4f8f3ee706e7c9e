// hz_ctx and the engine helpers shared by engine.cpp (NCCL transport) and
// p2p.cpp (NVLink peer-memory transport).  Internal header.
#pragma once

#include <nccl.h>

#include <string>
#include <vector>

#include "hz_internal.h"

struct hz_ctx {
  int rank = 0, world = 1, levels = 0, device = 0;
  int group[HZ_MAX_LEVELS] = {0};
  int digit[HZ_MAX_LEVELS] = {0};
  ncclComm_t world_comm = nullptr;
  ncclComm_t lvl[HZ_MAX_LEVELS] = {nullptr};
  struct Buf {
    void* p = nullptr;
    size_t cap = 0;
  };
  // NCCL transport workspace
  Buf ag_c, ag_s;                      // full-layer codes / scales (all-gather)
  Buf rs_a_c, rs_a_s, rs_b_c, rs_b_s;  // ping-pong send buffers (reduce-scatter)
  Buf rs_r_c, rs_r_s;                  // receive slots (reduce-scatter)
  Buf ar_a, ar_b, ar_g;                // allreduce + select: ping-pong fp32, gathered members

  // NVLink P2P transport (hz_enable_p2p): one IPC-mapped symmetric pool per rank.
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
    // prefetched quantize (hz_allgather_params_next): the next layer's primary was
    // quantized into pre_codes in phase pre_phase by the previous call's dual kernel
    unsigned long long pre_phase = 0;
    const void* pre_codes = nullptr;
    const void* pre_primary = nullptr;
    bool capturing = false;
    struct Slot {
      size_t off = 0, cap = 0;
    };
    Slot ag_prim_c, ag_prim_s;                  // quantized primary when s != w
    Slot rs_c[HZ_MAX_LEVELS + 1], rs_s[HZ_MAX_LEVELS + 1];   // level-l send buffers
    Slot upd;                                   // updated weights of range_L (step tail)
    Slot ar_a, ar_b;                            // allreduce + select: ping-pong fp32 buffers
    // push mode: receive buffers the producers store into over NVLink
    Slot ag_recv_c, ag_recv_s;                  // forward gather: D pieces of the primary codes
    Slot rs_recv_c[HZ_MAX_LEVELS + 1], rs_recv_s[HZ_MAX_LEVELS + 1];   // level-l: g chunks destined here
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

// header of the symmetric pool: ready[8] u64 | done[8] u64 | counter u32 | epoch u64 |
// pipelined-kernel ticket counters | per-chunk flags of the pipelined all-gather
// [8][kMaxChunks] and reduce-scatter [16][kMaxChunks] | per-chunk producer arrival
// counters (u32 [kMaxChunks] each)
constexpr size_t kReadyOff = 0, kDoneOff = 64, kCounterOff = 128, kEpochOff = 192;
constexpr size_t kWorkAGOff = 256, kWorkRSOff = 320;
constexpr size_t kChunkAGOff = 4096;
constexpr size_t kChunkRSOff = kChunkAGOff + size_t(kMaxWorld) * kMaxChunks * 8;
constexpr size_t kCntAGOff = kChunkRSOff + size_t(kMaxG) * kMaxChunks * 8;
constexpr size_t kCntRSOff = kCntAGOff + size_t(kMaxChunks) * 4;
constexpr size_t kDbgOff = kCntRSOff + size_t(kMaxChunks) * 4;   // HZ_TUNE pdbg timelines [kMaxChunks][4]
constexpr size_t kPoolHeader = kDbgOff + size_t(kMaxChunks) * 32;

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
// push kernels (P2P): `remote` = bytes stored into peer memory per launch
hz_status run_quantize_push(const void* x, hz_dtype dt, int64_t n, int bits, uint8_t* c, float* s, void* y,
                            hz_dtype odt, const PushDst& dst, cudaStream_t st, int level, const SyncArgs* sync,
                            int64_t remote);
hz_status run_reduce_push(int g, const uint8_t* const* c, const float* const* s, int64_t n, int bits_in,
                          int bits_out, const PushDst& dst, cudaStream_t st, int level, const SyncArgs* sync,
                          int64_t remote);
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
void exec_release(hz_ctx* ctx);   // executor.cpp
hz_status p2p_adamw_gather(hz_ctx* ctx, const hz_partition_t* p, const float* g, float* th, float* m, float* v,
                           const AdamW& hp, void* primary, hz_dtype dt, cudaStream_t st);
hz_status run_adamw(const float* g, float* th, float* m, float* v, void* out, hz_dtype dt, int64_t n,
                    const AdamW& hp, cudaStream_t st, const SyncArgs* sync);

}  // namespace hz
