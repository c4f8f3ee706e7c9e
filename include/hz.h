/*
 * hz.h — C ABI of libhz.so: the data-parallel hot path of hierarchical ZeRO++
 * (arXiv 2501.04266, "Scaling Large Language Model Training on Frontier with
 * Low-Bandwidth Partitioning") for NVIDIA B200 (sm_100a).
 *
 * Citations: P:<n> = line n of the paper's PAPER.md; S:<n> = line n of SPEC.md;
 * O<k>/R<k> = oracle step / reading, listed in DESIGN.md §3.
 *
 * What the library computes (per layer, per rank):
 *   - qwZ: block-quantize the rank's primary bf16/fp16/fp32 weight shard to
 *     int8 codes + one fp32 scale per block, all-gather the
 *     codes level by level inside the hierarchy (Table VII),
 *     keep the quantized secondary partition (hpZ, Table V) and
 *     dequantize the full layer.  Backward: gather again from the secondary.
 *   - qgZ: block-quantize the gradient to int4/int8 and reduce-scatter it as a
 *     hierarchical all-to-all, dequantizing and summing at each level
 *     (Table VIII), ending in an fp32 gradient shard.
 *
 * Hierarchy: g = (g_1..g_L), innermost level first, prod(g) = world.  Ranks are
 * numbered node-major: r = sum_l d_l(r) * prod_{k<l} g_k (O1).  Level l's
 * exchange group = the g_l ranks that differ only in digit d_l.  A level may
 * have g_l = 1 (no exchange; a one-GPU run uses g = (1)).
 *
 * Ownership map (O3, "digit-reversed"): off_0 = 0, len_0 = Np;
 * len_l = len_{l-1}/g_l, off_l = off_{l-1} + d_l*len_l.  Role levels:
 * primary weights = range_w, secondary = range_s, gradient = range_gl,
 * optimizer = range_L.  Nesting range_L c range_gl c range_w is the paper's
 * dependency rule N >= N_os >= N_g >= N_w.
 *
 * Codec (O4-O6, readings R1-R5): blocks of `block` contiguous elements;
 *   am = max|x|; am < 2^-100 -> scale 0, codes 0; else
 *   scale = fl32(am/qmax), inv = fl32(qmax/am),
 *   code = clamp(rne(fl32(x*inv)), -qmax, qmax), qmax = 127 (int8) / 7 (int4);
 *   x_hat = fl32(code*scale); bf16/fp16 output = RNE(x_hat).
 *   Reduction (O9): acc = x_hat_0; acc = fl32(acc + x_hat_p) for p = 1..g-1 in
 *   ascending level digit (no FMA); accumulate: A = fl32(A + acc).
 * Code layout: one codes array (int8: 1 byte/element, two's complement;
 * int4: 2 elements/byte, even element in the low nibble) and one fp32 scales
 * array, block k at index k ("SoA").  Every level chunk is therefore a
 * contiguous slice of both arrays.
 *
 * Conventions for every entry point:
 *   - Device pointers are CUDA device (or managed) pointers on the current /
 *     context device; they must be 16-byte aligned.  The caller allocates and
 *     owns every pointer it passes; the library owns its NCCL communicators and
 *     internal workspace (grown on first use to the largest layer seen; the
 *     growth call synchronises the device, so do one warm-up call per size).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     All device work is enqueued on it; calls return once enqueued
 *     (asynchronous).  Host-side validation is synchronous.
 *   - Return value: HZ_OK, or an error code with a message naming the offending
 *     argument available from hz_last_error() (thread-local).  Nothing is
 *     enqueued when validation fails.
 *   - Collective calls (hz_init, hz_allgather_params, hz_allgather_params_next,
 *     hz_reduce_scatter_grads, hz_backward_step, hz_allreduce_select,
 *     hz_adamw_step, hz_step_host, hz_finalize) must be issued by every rank in
 *     the same order with the same arguments' shapes (NCCL rule).
 *   - Non-finite inputs are a precondition violation; results are
 *     unspecified for them.
 */
#ifndef HZ_H_
#define HZ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define HZ_API __attribute__((visibility("default")))
#else
#define HZ_API
#endif

#define HZ_MAX_LEVELS 4

typedef struct hz_ctx hz_ctx; /* opaque: device, NCCL comms per level, workspace */

typedef enum {
  HZ_OK = 0,
  HZ_ERR_INVALID = 1,     /* bad argument; message names the field */
  HZ_ERR_CUDA = 2,        /* CUDA runtime / launch error */
  HZ_ERR_NCCL = 3,        /* NCCL error (incl. asynchronous errors of earlier calls) */
  HZ_ERR_NONFINITE = 4,   /* reserved for debug builds */
  HZ_ERR_UNSUPPORTED = 5, /* valid request this build does not implement */
  HZ_ERR_ABORTED = 6      /* the context was aborted (a cross-GPU wait timed out, or
                             hz_abort); only hz_finalize is allowed afterwards */
} hz_status;

typedef enum { HZ_F32 = 0, HZ_BF16 = 1, HZ_F16 = 2 } hz_dtype;

typedef struct { unsigned char bytes[128]; } hz_uid; /* = ncclUniqueId */

/* Per-rank partition of one flat per-layer buffer (O1-O3). */
typedef struct {
  int64_t numel;         /* logical element count n */
  int64_t padded_numel;  /* Np = ceil(n / (world*4*block)) * world*4*block (O2, zero pad) */
  int32_t block;         /* quantization block B */
  int32_t levels;        /* L */
  int32_t world;         /* prod(group) */
  int32_t rank;
  int32_t w, s, gl;      /* role levels: primary, secondary, gradient (0..L) */
  int32_t group[HZ_MAX_LEVELS];  /* g_l, l = 1..L at index l-1 */
  int32_t digit[HZ_MAX_LEVELS];  /* d_l(rank) at index l-1 */
  int64_t off[HZ_MAX_LEVELS + 1];/* off_l, l = 0..L (elements) */
  int64_t len[HZ_MAX_LEVELS + 1];/* len_l, l = 0..L (elements) */
  /* qgZ hop grouping ("1-hop all-to-all", reading R15): the reduce-scatter
   * runs one all-to-all per hop; hop k covers levels hop_last[k-1]+1 .. hop_last[k]
   * (hop_last[-1] = 0).  nhops == 0: one hop per level (the default written by
   * hz_partition / hz_partition_ex).  Set with hz_partition_set_hops. */
  int32_t nhops;
  int32_t hop_last[HZ_MAX_LEVELS];
} hz_partition_t;

/* Library version string, e.g. "hz 0.1 sm_100a". Never NULL. */
HZ_API const char* hz_version(void);

/* Message of the last non-OK status returned on this thread ("" if none). */
HZ_API const char* hz_last_error(void);

/* Number of exported entry points and their names (for ABI checks). */
HZ_API int hz_num_symbols(void);
HZ_API const char* hz_symbol_name(int i);

/* ---------------------------------------------------------------- host only */

/* O1-O3 (Table IV).  Pure host function; needs no GPU.
 * rank in [0, prod(group)); levels in [1, HZ_MAX_LEVELS]; group[l] >= 1;
 * numel >= 0; block a power of two in [32, 2048]; 0 <= w, s, gl <= levels.
 * Writes *out.  Errors: HZ_ERR_INVALID. */
HZ_API hz_status hz_partition_ex(int rank, int levels, const int* group, int64_t numel,
                          int block, int w, int s, int gl, hz_partition_t* out);

/* Merged-level qgZ (the 1-hop all-to-all reduce-scatter; "the
 * hop grouping is a parameter"; reading R15).  Sets p's hop grouping: nhops in
 * [1, levels], hop_last strictly ascending, hop_last[nhops-1] == levels; nhops == 0
 * (hop_last ignored) restores one hop per level.  A hop over levels a..b is ONE
 * all-to-all over the prod_{l=a..b} g_l ranks that share every digit outside a..b:
 * the member whose digits are (d_a..d_b) receives the chunk of range_{a-1} at
 * sum_{l=a..b} d_l*len_l (its range_b — the ownership map is unchanged, O3), and
 * each rank sums the members' dequantized chunks in ascending rank order, fp32, no
 * FMA.  One quantization per hop: fewer requantizations than per-level hops (the
 * error P:122 designs against), more peers per all-to-all.  Every qgZ entry point
 * (hz_reduce_scatter_grads, hz_backward_step, hz_step_host) and
 * hz_plan_reduce_scatter follow the grouping; their from_level / to_level must fall
 * on hop boundaries.  Pure host function.  Errors: HZ_ERR_INVALID. */
HZ_API hz_status hz_partition_set_hops(hz_partition_t* p, int nhops, const int* hop_last);

/* Communication plan of one rank: the exact NCCL operations hz_allgather_params /
 * hz_reduce_scatter_grads issue, in order (the engine issues its calls from
 * these plans).  Pure host functions; used by the CPU (gloo) tests to check
 * that every send matches a receive on the peer.
 *   HZ_PLAN_ALLGATHER: level-l all-gather of this rank's piece range_l
 *     (send_off, elems) into range_{l-1} (recv_off), over the g_l members;
 *     all-gather top = w (forward) or s (backward) down to 1, levels with
 *     g_l = 1 omitted (O7/O8, Table VII).
 *   HZ_PLAN_SENDRECV: exchange of the hop over levels level..level_last with
 *     the member of merged digit `peer` (global rank peer_rank; its index in
 *     ascending rank order within the hop group): send that member's chunk of
 *     range_{level-1} (send_off, elems) and receive its chunk for range_{level_last}
 *     (recv_off); peers in ascending merged digit, hops from..to (O9, Table
 *     VIII).  With one hop per level, level_last == level and peer is the level
 *     digit.
 * Offsets are global element offsets of the padded layer; code_bytes /
 * scale_bytes are the bytes of one piece / chunk.  *n_out = number of steps
 * (all of them, even when max is smaller; copies min(max, n)). */
typedef enum { HZ_PLAN_ALLGATHER = 1, HZ_PLAN_SENDRECV = 2 } hz_plan_op;

typedef struct {
  int32_t op;         /* hz_plan_op */
  int32_t level;      /* 1..L (SENDRECV: first level of the hop) */
  int32_t level_last; /* SENDRECV: last level of the hop; ALLGATHER: == level */
  int32_t group;      /* members of the exchange (g_level, or the hop's product) */
  int32_t peer;       /* SENDRECV: peer's level digit (its level-communicator rank); else -1 */
  int32_t peer_rank;  /* SENDRECV: peer's global rank; else -1 */
  int32_t bits;       /* code width */
  int64_t elems;
  int64_t send_off;
  int64_t recv_off;
  int64_t code_bytes;
  int64_t scale_bytes;
} hz_comm_step;

HZ_API hz_status hz_plan_allgather(const hz_partition_t* p, int backward, int bits,
                                   hz_comm_step* out, int max, int* n_out);
HZ_API hz_status hz_plan_reduce_scatter(const hz_partition_t* p, int from_level, int to_level,
                                        const int* bits_per_level, hz_comm_step* out, int max,
                                        int* n_out);

/* ------------------------------------------------------- standalone codec ops */

/* O4: quantize x[0..n) (dtype dt) into codes (n*bits/8
 * bytes) and scales (n/block fp32).  n % block == 0; bits in {4, 8};
 * block a power of two in [32, 2048].  n == 0 is a no-op. */
HZ_API hz_status hz_quantize(const void* x, hz_dtype dt, int64_t n, int bits, int block,
                      uint8_t* codes, float* scales, void* stream);

/* O6: y[0..n) = dtype(out_dt)(fl32(code * scale)); same constraints as hz_quantize. */
HZ_API hz_status hz_dequantize(const uint8_t* codes, const float* scales, int64_t n, int bits,
                        int block, void* y, hz_dtype out_dt, void* stream);

/* O9 level step (A9): g inputs (host array of g device pointer pairs, input p =
 * the chunk from the member with level digit p, each n elements coded with
 * bits_in), summed in ascending p in fp32 without FMA.  Exactly one output:
 *   bits_out in {4, 8}: requantize the sum into out_codes / out_scales (the
 *                       next level's send layout = this chunk's SoA arrays);
 *   bits_out == 0:      write fp32 out_f32[0..n) (accumulate != 0: += ).
 * 1 <= g <= 16. */
HZ_API hz_status hz_reduce_chunks(int g, const uint8_t* const* codes, const float* const* scales,
                           int64_t n, int bits_in, int block, int bits_out,
                           uint8_t* out_codes, float* out_scales, float* out_f32,
                           int accumulate, void* stream);

/* ------------------------------------------------------------- collectives */

/* A fresh ncclUniqueId; call on one rank and broadcast the 128 bytes. */
HZ_API hz_status hz_get_uid(hz_uid* out);

/* Collective over all `world` ranks.  Selects `cuda_device`, creates the world
 * NCCL communicator and, with ncclCommSplit(color = rank - d_l*stride_l,
 * key = d_l), one communicator per level with g_l > 1.  levels in
 * [1, HZ_MAX_LEVELS], prod(group) == world.  workspace_bytes: optional
 * pre-reservation (0 = grow on first use).  *out owns everything it creates. */
HZ_API hz_status hz_init(hz_ctx** out, int rank, int world, const hz_uid* uid, int levels,
                  const int* group, int cuda_device, size_t workspace_bytes);

/* Destroys the communicators and frees the workspace.  NULL is a no-op.  CUDA graphs
 * that captured this context's NCCL-transport calls must be destroyed first (NCCL
 * keeps graph-owned resources on the communicators; destroying them under a live
 * graph blocks). */
HZ_API hz_status hz_finalize(hz_ctx* ctx);

/* hz_partition_ex for the context's rank and hierarchy. */
HZ_API hz_status hz_partition(const hz_ctx* ctx, int64_t numel, int block, int w, int s, int gl,
                       hz_partition_t* out);

/* qwZ + hpZ all-gather (O7 forward, O8 backward; Table VII).
 *   backward == 0: quantize primary (dt[len_w], the rank's range_w; NULL not
 *     allowed) with `bits`, all-gather levels w..1 (in place, per level
 *     communicator), write the secondary codes/scales of range_s to
 *     sec_codes (len_s*bits/8 bytes) / sec_scales (len_s/block fp32), and
 *     dequantize all of [0, Np) into full_out (out_dt[Np]).
 *   backward != 0: primary ignored (may be NULL); all-gather from the
 *     secondary over levels s..1 and dequantize into full_out.  The result is
 *     bitwise equal to the forward result (O8).
 * Padding elements [numel, Np) of the primary must be zero (O2). */
HZ_API hz_status hz_allgather_params(hz_ctx* ctx, const hz_partition_t* p, int backward,
                              const void* primary, hz_dtype dt, int bits,
                              uint8_t* sec_codes, float* sec_scales,
                              void* full_out, hz_dtype out_dt, void* stream);

/* Forward gather with the next layer's quantize prefetched (qwZ, same result as
 * hz_allgather_params forward for layer p): the gather + dequantize of layer p and
 * the quantize of layer p_next's primary (next_primary, dt[len_w of p_next]) into its
 * secondary buffers (next_sec_codes / next_sec_scales, int8 codes + fp32 scales of
 * range_s) run in ONE kernel (P2P transport: the NVLink-bound gather and the
 * HBM-bound quantize overlap; one launch and one cross-GPU synchronisation fewer).
 * The next call for layer p_next (hz_allgather_params or _next, with the same primary
 * and secondary pointers, and no other collective call in between) then skips its
 * quantize.  The caller must not modify next_primary in between.  p_next == NULL:
 * exactly hz_allgather_params(forward).  Not fusable (NCCL transport, s != w, block
 * != 256, bits != 8, out_dt != bf16): the prefetch is skipped and the next call
 * quantizes itself — results are bitwise identical either way.  Errors as
 * hz_allgather_params; p_next / next_* fields are named in the message. */
HZ_API hz_status hz_allgather_params_next(hz_ctx* ctx, const hz_partition_t* p, const void* primary, hz_dtype dt,
                                          int bits, uint8_t* sec_codes, float* sec_scales, void* full_out,
                                          hz_dtype out_dt, const hz_partition_t* p_next, const void* next_primary,
                                          uint8_t* next_sec_codes, float* next_sec_scales, void* stream);

/* Backward step of a layer pair: the qgZ reduce-scatter of layer p's gradient
 * (exactly hz_reduce_scatter_grads with the same arguments) and the backward
 * all-gather of the previous layer p_prev from its secondary (exactly
 * hz_allgather_params(backward = 1, bits = prev_bits) into prev_full_out) — the
 * order a training step issues them in (layer i's gradients are reduced while layer
 * i-1's weights are gathered for its backward).  P2P transport, B = 256, bf16
 * output: the gather and the level-`from` quantize run in ONE kernel; otherwise the
 * gather then the reduce-scatter.  p_prev == NULL: exactly hz_reduce_scatter_grads.
 * Deferred last hop (P2P transport, B = 256, p_prev given): the last qgZ hop of layer
 * p (its fp32 shard) is not launched by this call but carried by the next call on the
 * context — the next hz_backward_step runs it in the same kernel as its own gather and
 * quantize (the backward triple kernel: one launch and one cross-GPU synchronisation
 * fewer per layer), any other call (or hz_flush) first launches it on its own.  So
 * `shard` holds layer p's result once the stream passes the NEXT call on this context
 * (a training step's last hz_backward_step, with p_prev == NULL, completes everything);
 * results are bitwise those of hz_reduce_scatter_grads.  HZ_TUNE defer=0 disables it. */
HZ_API hz_status hz_backward_step(hz_ctx* ctx, const hz_partition_t* p, const void* grad, hz_dtype dt,
                                  int from_level, int to_level, const int* bits_per_level, float* shard,
                                  int accumulate, const hz_partition_t* p_prev, uint8_t* prev_sec_codes,
                                  float* prev_sec_scales, int prev_bits, void* prev_full_out,
                                  hz_dtype prev_out_dt, void* stream);

/* qgZ hierarchical all-to-all reduce-scatter (O9; Table VIII).
 * grad: dt[len_{from_level-1}] over the rank's range_{from_level-1}
 *   (from_level == 1: the full padded gradient dt[Np]).
 * Levels from_level..to_level (1 <= from <= to <= L) run in order; level l
 * quantizes with bits_per_level[l-1] in {4, 8}, exchanges chunks with the g_l-1
 * peers (grouped ncclSend/ncclRecv; the self chunk never enters NCCL), and
 * dequantizes + sums (+ requantizes for the next level).
 * shard: fp32[len_to_level] over range_to_level; accumulate != 0: shard += sum.
 * Setting T (the paper's ZeRO-topo): per micro-batch from=1, to=gl with
 * accumulate; once per step from=gl+1, to=L on the accumulated shard. */
HZ_API hz_status hz_reduce_scatter_grads(hz_ctx* ctx, const hz_partition_t* p, const void* grad,
                                  hz_dtype dt, int from_level, int to_level,
                                  const int* bits_per_level, float* shard, int accumulate,
                                  void* stream);

/* A10, the paper-literal cross-node step ("call Allreduce ... select the
 * gradients matching the on-device optimizer states"; reading R12).
 * shard_in: fp32[len_{from_level-1}] over range_{from_level-1} (device, read only).
 * Levels from_level..to_level run in order; at level l every rank sums the g_l
 * members' buffers element by element in ascending level digit (fp32, one
 * rounding per add, unquantized) — an allreduce — and after the last level keeps
 * range_{to_level}: out = fp32[len_{to_level}] (device, caller-owned).  The result
 * is bitwise equal to oracle/collectives.allreduce_select and to an unquantized
 * reduce-scatter over the same levels; it moves (g_l - 1) * len_{from_level-1}
 * fp32 per level and rank, twice the reduce-scatter's bytes (the reason the
 * default cross-node step is hz_reduce_scatter_grads).  Collective; transports:
 * NCCL (all-gather per level communicator + ordered local sum) or P2P (peers'
 * buffers read in place).  Errors: HZ_ERR_INVALID (levels, NULL / misaligned
 * pointers), HZ_ERR_CUDA, HZ_ERR_NCCL. */
HZ_API hz_status hz_allreduce_select(hz_ctx* ctx, const hz_partition_t* p, const float* shard_in,
                                     int from_level, int to_level, float* out, void* stream);

/* NVLink peer-memory transport (collective over all ranks of the context; one
 * node, world <= 8).  Allocates this rank's symmetric pool of pool_bytes,
 * exchanges CUDA IPC handles over NCCL and maps every peer's pool.  Afterwards
 * hz_allgather_params / hz_reduce_scatter_grads run with the collective fused
 * into the codec kernels: the gather+dequantize kernel reads the members' codes
 * straight from their pools over NVLink and the level reduce reads the peers'
 * chunks in place (no NCCL on the data path); cross-GPU ordering uses per-phase
 * flags in the pools.  Results are bitwise identical to the NCCL transport.
 * Requirements in P2P mode: the hpZ secondary buffers passed to
 * hz_allgather_params must come from hz_sym_alloc; all calls of the context on
 * one stream.  HZ_ERR_UNSUPPORTED if a peer cannot be mapped. */
HZ_API hz_status hz_enable_p2p(hz_ctx* ctx, size_t pool_bytes);
HZ_API hz_status hz_p2p_enabled(const hz_ctx* ctx, int* out);

/* Virtual world: `world` contexts (ranks 0..world-1 of hierarchy `group`) in THIS
 * process on ONE GPU, with the P2P transport enabled and every rank's "peer" pool
 * being another context's allocation (pool_bytes each; no IPC, no NCCL).  The same
 * exchange kernels, flags and phase protocol run as on `world` GPUs; additionally
 * every synchronised launch is ordered on the host after the launches that signal
 * what it waits for (CUDA events), so the contexts must be driven concurrently from
 * one host thread each (one stream each), issuing the same call sequence per rank —
 * a call blocks its thread until the ranks it waits for have issued their side.
 * Intended for testing the multi-rank path on one GPU (tests/vworld.py).  Not
 * supported in a virtual world: NCCL-transport and flat calls, graph capture.
 * 1 <= world <= 8.  out: array of `world` context pointers; each is finalised with
 * hz_finalize (the pools are freed with the last one; finalise every context after
 * all their work, every context's thread must be done).  Errors: HZ_ERR_INVALID,
 * HZ_ERR_UNSUPPORTED (world > 8), HZ_ERR_CUDA. */
HZ_API hz_status hz_init_virtual(hz_ctx** out, int world, int levels, const int* group, int cuda_device,
                                 size_t pool_bytes);

/* hz_init_virtual with rank r's pool and kernels on GPU devices[r] (devices: `world`
 * ordinals; ranks on different GPUs read each other's pools over NVLink through peer
 * access, enabled here; HZ_ERR_UNSUPPORTED if two of the devices cannot map each
 * other).  Same protocol and host ordering as hz_init_virtual: every kernel starts
 * after the kernels it waits for have completed, so a profiler that serialises
 * launches (ncu) can replay the P2P exchange kernels of a real multi-GPU exchange
 * from one process (tools/vw_profile.py).  Each rank's thread must make devices[r]
 * current before calling into its context.  hz_init_virtual(..., d, ...) ==
 * hz_init_virtual_ex with devices[r] = d for every r. */
HZ_API hz_status hz_init_virtual_ex(hz_ctx** out, int world, int levels, const int* group, const int* devices,
                                    size_t pool_bytes);

/* Failure handling of the P2P transport.  A kernel waits for its peers'
 * phase flags at most `seconds` (default 600 s, so checkpoint saves or evaluation on
 * one rank do not break the others); a longer wait, or hz_abort (from any host thread,
 * e.g. a watchdog), aborts the context: every waiting kernel returns without work or
 * signals (no sticky CUDA error, no hung GPU) and every later call except hz_finalize
 * returns HZ_ERR_ABORTED.  Peers of an aborted rank time out in turn.  hz_check
 * returns HZ_ERR_ABORTED / HZ_ERR_NCCL (asynchronous errors of any of the context's
 * NCCL communicators, which are then aborted) or HZ_OK without enqueuing anything. */
HZ_API hz_status hz_set_wait_timeout(hz_ctx* ctx, double seconds);

/* Measurement helper (bench.py's NVLink roofline denominator):
 * reads `bytes` (a multiple of 16, within the pool) of rank `peer`'s symmetric pool
 * `reps` times with the load path of the fused gather / reduce kernels (16-byte
 * coherent loads, a full grid) on `stream`, after one warm-up read, and writes the
 * average milliseconds per read to *ms_out (synchronises the stream).  Not a
 * collective: run it on several ranks at once (after a barrier) to measure both
 * directions of a link loaded together.  Errors: HZ_ERR_INVALID, HZ_ERR_CUDA. */
HZ_API hz_status hz_nvlink_probe(hz_ctx* ctx, int peer, size_t bytes, int reps, float* ms_out, void* stream);
HZ_API hz_status hz_abort(hz_ctx* ctx);
/* Complete deferred work of the P2P transport on `stream`: a deferred last qgZ hop of
 * hz_backward_step and the phase of a prefetched quantize of hz_allgather_params_next
 * (a later call does this implicitly).  Collective: every rank issues it at the same
 * point of the call sequence.  No-op without the P2P transport or pending work.
 * Errors: HZ_ERR_INVALID (ctx NULL), HZ_ERR_ABORTED, HZ_ERR_CUDA. */
HZ_API hz_status hz_flush(hz_ctx* ctx, void* stream);
HZ_API hz_status hz_check(const hz_ctx* ctx);

/* CUDA-graph support for the P2P transport.  The cross-GPU phase numbers are
 * stored in the kernels relative to a device-side epoch, so a captured step can
 * be replayed: bracket the capture of one step with hz_p2p_capture_begin /
 * hz_p2p_capture_end (the latter appends a one-thread node that advances the
 * epoch by the step's phase count, returned in *span_out), and after launching
 * the graph n times call hz_p2p_replayed(ctx, n) so that later eager calls
 * continue the numbering.  Every rank must capture and replay identically. */
HZ_API hz_status hz_p2p_capture_begin(hz_ctx* ctx);
HZ_API hz_status hz_p2p_capture_end(hz_ctx* ctx, void* stream, unsigned long long* span_out);
HZ_API hz_status hz_p2p_replayed(hz_ctx* ctx, unsigned long long n);

/* Symmetric allocation from the P2P pool (256-byte aligned).  Every rank must make
 * the same sequence of calls with the same sizes, so that a buffer has the same
 * pool offset on every rank.  Freed with the context.  HZ_ERR_INVALID when the pool
 * is exhausted or P2P is not enabled. */
HZ_API hz_status hz_sym_alloc(hz_ctx* ctx, size_t bytes, void** out);

/* Step tail: AdamW on the rank's optimizer shard followed by
 * the post-update all-gather of the updated weights.
 * grad_shard, master, m, v: fp32[len_L] over range_L (master / m / v updated in
 * place).  primary: dt[len_w] over range_w, overwritten with the updated weights
 * of range_w (its range_L part from this rank's update, the rest gathered from
 * the ranks that share digits 1..w, over levels L..w+1; no quantization — the
 * narrow form of P:399's exchange allowed by the nested ownership map).
 * Arithmetic (reading R19, PyTorch AdamW, fp32, one rounding per operation):
 *   m' = b1*m + omb1*g;  v' = b2*v + (omb2*g)*g;  th1 = th - lr_wd*th;
 *   th' = th1 - step * (m' / (sqrt(v')/sqrt_bc2 + eps));  primary = dt(th')
 * with the host scalars of hz_adamw_t (omb = 1 - b, lr_wd = lr*wd,
 * sqrt_bc2 = sqrt(1 - b2^t), step = lr / (1 - b1^t)). */
typedef struct {
  float b1, omb1, b2, omb2, lr_wd, sqrt_bc2, eps, step;
} hz_adamw_t;
/* The hz_adamw_t of step t >= 1 (reading R19): every constant computed in double
 * and rounded once to fp32 (omb1 = 1-b1, omb2 = 1-b2, lr_wd = lr*weight_decay,
 * sqrt_bc2 = sqrt(1-b2^t), step = lr/(1-b1^t)).  Pure host function.
 * Errors: HZ_ERR_INVALID (NULL out, t < 1, b1 / b2 outside [0, 1)). */
HZ_API hz_status hz_adamw_params(double lr, double b1, double b2, double eps, double weight_decay, int64_t t,
                                 hz_adamw_t* out);
HZ_API hz_status hz_adamw_step(hz_ctx* ctx, const hz_partition_t* p, const float* grad_shard,
                               float* master, float* m, float* v, const hz_adamw_t* hp,
                               void* primary, hz_dtype dt, void* stream);

/* Host-staged step executor: one step of the hot path with its inputs and results
 * in HOST memory (the end-to-end form of SURVEY §8(d)'s step; the per-layer phase
 * order of P:275 / S:359 with one micro-batch, GA = 1).  For n tensors t[0..n-1]:
 *   forward : i = 0..n-1   copy t[i].h_primary -> t[i].d_primary (dt[len_w]),
 *                          hz_allgather_params(forward, qwz_bits) -> full_out[i % 2];
 *   backward: i = n-1..0   copy t[i].h_grad -> t[i].d_grad (dt[Np]),
 *                          hz_allgather_params(backward) -> full_out[i % 2],
 *                          hz_reduce_scatter_grads(levels 1..L, qgz_bits) -> t[i].d_shard,
 *                          copy t[i].d_shard -> t[i].h_shard (fp32[len_L]).
 * The kernels are issued as the paired calls of a training step
 * (hz_allgather_params_next with layer i+1 as next; hz_backward_step with layer i-1
 * as prev), so on the P2P transport adjacent layers share launches; the results are
 * those of the single calls above, bitwise.
 * The copies run on two library-owned streams (host->device and device->host), the
 * kernels on `stream`; per-tensor events order them, so the PCIe transfers of the
 * two directions overlap each other and the kernels.  `stream` finally waits for
 * every device->host copy: once `stream` passes this call, every h_shard holds the
 * step's fp32 gradient shard (bitwise the result of the device-resident calls).
 * The host->device copies of a call wait only for the previous call's kernels, so
 * back-to-back calls upload the next step's inputs while this step's shards are
 * still being read back.
 * Ownership: the caller owns every buffer.  h_* should be page-locked
 * (cudaHostAlloc / cudaHostRegister) for the copies to be asynchronous; they must
 * not be modified (h_primary, h_grad) or read (h_shard) before `stream` passes the
 * call.  d_primary / d_grad are staging buffers owned by the executor from the first
 * call on: the caller must not read or write them on any stream, `stream` included,
 * between calls (the next call's uploads into them start as soon as the previous
 * call's kernels are done, without waiting for other work on `stream`).  sec_codes / sec_scales: the hpZ
 * secondary of range_s (P2P transport: from hz_sym_alloc).  full_out0/1: device
 * out_dt[max Np] gathered-layer buffers, alternating between tensors.
 * Errors: HZ_ERR_INVALID (n < 1, NULL pointers, a partition of another context or
 * with an invalid block / padding / hop grouping, misaligned device pointers, P2P
 * transport: secondaries outside the symmetric pool; message names the tensor and
 * field; nothing is enqueued), HZ_ERR_CUDA, HZ_ERR_NCCL; errors of the underlying calls are passed
 * through (work already enqueued for earlier tensors stays enqueued). */
typedef struct {
  const hz_partition_t* p;
  const void* h_primary; /* host dt[len_w] (range_w) */
  void* d_primary;       /* device dt[len_w] */
  const void* h_grad;    /* host dt[Np] */
  void* d_grad;          /* device dt[Np] */
  uint8_t* sec_codes;    /* device, range_s codes (len_s*qwz_bits/8 bytes) */
  float* sec_scales;     /* device, range_s scales (len_s/block fp32) */
  float* d_shard;        /* device fp32[len_L] */
  float* h_shard;        /* host fp32[len_L] */
} hz_tensor_io;
HZ_API hz_status hz_step_host(hz_ctx* ctx, int n, const hz_tensor_io* t, hz_dtype dt, int qwz_bits,
                              const int* qgz_bits, void* full_out0, void* full_out1, hz_dtype out_dt,
                              void* stream);

/* Flat ZeRO-3 baseline (Table VII/VIII row "ZeRO-3"): plain ncclAllGather of
 * the rank's bf16/fp16/fp32 chunk (numel/world elements, rank order) into
 * out[numel], and plain ncclReduceScatter(sum) of in[numel] into
 * out_chunk[numel/world].  numel % world == 0. */
HZ_API hz_status hz_flat_allgather(hz_ctx* ctx, const void* chunk, void* out, int64_t numel,
                            hz_dtype dt, void* stream);
HZ_API hz_status hz_flat_reduce_scatter(hz_ctx* ctx, const void* in, void* out_chunk,
                                 int64_t numel, hz_dtype dt, void* stream);

/* SM budget of every libhz kernel launch (process-wide; 0 = all SMs, the default).
 * Grids are sized to `sms` x the kernel's resident CTAs per SM instead of the whole
 * GPU.  All kernels are grid-stride loops, so any budget is correct.  Intended for
 * communication streams confined to an SM partition (a CUDA green context of
 * `sms` SMs) while compute kernels run on the rest (tools/train_step.py --green).
 * Errors: HZ_ERR_INVALID if sms < 0. */
HZ_API hz_status hz_set_sm_budget(int sms);

/* ------------------------------------------------------------------ tracing */

/* Per-launch device timing of the library's own work: CUDA events around each
 * kernel / NCCL group on its stream and/or in-kernel device-clock stamps.
 * hz_trace_begin(cap, flags) starts recording up to cap records of the calling
 * host thread's launches (per thread, so that the contexts of a virtual world, one
 * thread each, trace separately); hz_trace_end() stops.  hz_trace_read
 * synchronises the recorded events and copies up to max records.  kind is a
 * static string ("quantize", "dequantize", "reduce", "reduce_requant",
 * "nccl_allgather", "nccl_alltoall", "nccl_flat", "copy"). bytes = algorithmic
 * HBM bytes (kernels) or bytes sent per rank (NCCL). */
typedef struct {
  const char* kind;
  int32_t level;
  int32_t bits;
  int64_t elems;
  int64_t bytes;        /* algorithmic bytes of this GPU's HBM (kernels) / bytes sent (NCCL) */
  int64_t remote_bytes; /* P2P kernels: bytes read from peers over NVLink; else 0 */
  float ms;        /* CUDA-event duration of the launch on its stream */
  float wait_ms;   /* P2P kernels: time CTA 0 spent waiting for peers (device clock); else -1 */
  float work_ms;   /* P2P kernels: after-wait to last CTA arrival (device clock); else -1 */
  float publish_ms;/* P2P kernels: last CTA's fence + flag stores (device clock); else -1 */
  float stamp_ms;  /* kernels, HZ_TRACE_STAMPS: CTA 0 entry to the last CTA's exit, including
                      the P2P flag publication (device clock); else -1 */
} hz_trace_rec;

#define HZ_TRACE_EVENTS 1  /* CUDA event pair around every launch (adds stream operations) */
#define HZ_TRACE_STAMPS 2  /* in-kernel %globaltimer stamps (no stream operations; kernels only) */
HZ_API hz_status hz_trace_begin(int capacity, int flags);
HZ_API hz_status hz_trace_end(void);
HZ_API hz_status hz_trace_read(hz_trace_rec* out, int max, int* n_out);

#ifdef __cplusplus
}
#endif

#endif /* HZ_H_ */
