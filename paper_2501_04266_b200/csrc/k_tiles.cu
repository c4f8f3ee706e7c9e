// The TMA tile-engine kernels (tiles.cuh): quantize (A2 / A7), the fused round trip of a
// one-member level, gather+dequantize (A3 / A5 / A6, pieces local or over NVLink), the
// dual gather || quantize launch, and the level reduce (A9 / A10).  Same arithmetic and
// order as the LSU kernels (k_quantize.cu, k_dequantize.cu, k_reduce.cu), so the outputs
// are bitwise identical.  Off by default (HZ_TUNE tma=1 enables it; measured slower,
// tiles.cuh); when on, the LSU kernels still take the shapes the engine does not
// (block != 256, lengths not a multiple of 1024, unaligned buffers, the accumulating
// round trip).
#include "tiles.cuh"

namespace hz {
namespace {

using namespace dev;

template <class Job>
__global__ void __launch_bounds__(kThreads, 4) k_tiles(const __grid_constant__ Job job, TileGeo geo,
                                                       const __grid_constant__ SyncArgs sy) {
  extern __shared__ __align__(128) char smem[];
  if (!sync_wait(sy)) return;
  const Pipe p = pipe_init(smem, geo);
  run_tiles(job, p, blockIdx.x, gridDim.x);
  sync_signal(sy);
}

int up128(int b) { return (b + 127) / 128 * 128; }

// te (elements per tile) and S (input stages) for in(te) / out(te) bytes: the largest of
// te = HZ_TUNE tte (default 8192) halving down to 1024, S = HZ_TUNE ts (default 3) down to
// 2, within the shared-memory budget of 3 CTAs per SM (HZ_TUNE tsm, bytes).  Measured
// (tools/tma_mix_probe.cu): 8192-element tiles with 2-3 stages are the fastest for every
// byte mix of the codec (larger bulk copies; 3-4 CTAs per SM keep them in flight).
template <class In, class Out>
TileGeo pick(In in, Out out) {
  static const int te0 = tune_param("tte", 8192);
  static const int s0 = tune_param("ts", 3);
  static const int budget = tune_param("tsm", 74 * 1024);
  TileGeo g{};
  for (int te = te0; te >= 1024; te /= 2) {
    for (int S = s0; S >= 2; --S) {
      g = TileGeo{te, S, up128(in(te)), up128(out(te))};
      if (g.smem() <= budget) return g;
    }
  }
  return TileGeo{1024, 2, up128(in(1024)), up128(out(1024))};
}

template <class Job>
cudaError_t launch_job(const Job& job, const TileGeo& g, int64_t ntiles, cudaStream_t st, const SyncArgs& sy) {
  auto kern = k_tiles<Job>;
  const int64_t grid = grid_for(reinterpret_cast<const void*>(kern), ntiles * (kThreads / 32), g.smem());
  return launch_k_smem(kern, grid, g.smem(), st, job, g, sy);
}

bool a16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ------------------------------------------------------------------------ quantize
template <typename T, int BITS, int OUT>
cudaError_t quant_t(const void* x, int64_t n, uint8_t* codes, float* scales, void* y, cudaStream_t st,
                    const SyncArgs& sy) {
  using J = QuantJob<T, BITS, OUT>;
  const bool hc = codes != nullptr;
  const TileGeo g = pick([](int te) { return J::in_bytes(te); }, [hc](int te) { return J::out_bytes(te, hc); });
  J job{static_cast<const T*>(x), n, codes, scales, static_cast<typename J::TO*>(y), g.te};
  return launch_job(job, g, (n + g.te - 1) / g.te, st, sy);
}

template <typename T, int BITS>
cudaError_t quant_o(const void* x, int64_t n, uint8_t* codes, float* scales, void* y, int out, cudaStream_t st,
                    const SyncArgs& sy) {
  switch (out) {
    case 0: return quant_t<T, BITS, 0>(x, n, codes, scales, y, st, sy);
    case 1: return quant_t<T, BITS, 1>(x, n, codes, scales, y, st, sy);
    case 2: return quant_t<T, BITS, 2>(x, n, codes, scales, y, st, sy);
    case 3: return quant_t<T, BITS, 3>(x, n, codes, scales, y, st, sy);
  }
  return cudaErrorInvalidValue;
}

int out_code(int has_y, hz_dtype out_dt) {
  if (!has_y) return 0;
  return out_dt == HZ_BF16 ? 1 : out_dt == HZ_F16 ? 2 : 3;
}

// -------------------------------------------------------------------------- gather
template <int BITS, typename TO>
GatherJob<BITS, TO> gather_job(const Pieces& pc, void* y, int te) {
  GatherJob<BITS, TO> j{};
  j.pc = pc;
  j.y = static_cast<TO*>(y);
  j.te = te;
  j.tpp = (pc.len + te - 1) / te;
  return j;
}

template <int BITS, typename TO>
cudaError_t gather_t(const Pieces& pc, void* y, cudaStream_t st, const SyncArgs& sy) {
  using J = GatherJob<BITS, TO>;
  const bool hs = pc.sec_c != nullptr;
  const TileGeo g = pick([](int te) { return J::in_bytes(te); }, [hs](int te) { return J::out_bytes(te, hs); });
  const J job = gather_job<BITS, TO>(pc, y, g.te);
  return launch_job(job, g, job.tpp * pc.n, st, sy);
}

// ---------------------------------------------------------------------------- dual
template <typename T, int QBITS, int QOUT>
cudaError_t dual_t(const Pieces& pc, void* y, const void* x, int64_t nq, uint8_t* codes, float* scales, float* qy,
                   cudaStream_t st, const SyncArgs& sy) {
  using GJ = GatherJob<8, __nv_bfloat16>;
  using QJ = QuantJob<T, QBITS, QOUT>;
  const bool hs = pc.sec_c != nullptr, hc = codes != nullptr;
  const TileGeo g = pick([](int te) { return std::max(GJ::in_bytes(te), QJ::in_bytes(te)); },
                         [hs, hc](int te) { return std::max(GJ::out_bytes(te, hs), QJ::out_bytes(te, hc)); });
  DualJob<GJ, QJ> job{gather_job<8, __nv_bfloat16>(pc, y, g.te),
                      QJ{static_cast<const T*>(x), nq, codes, scales, qy, g.te}};
  return launch_job(job, g, job.g.tpp * pc.n + (nq + g.te - 1) / g.te, st, sy);
}

// -------------------------------------------------------------------------- reduce
template <int BIN, int GT, int MODE, int BOUT>
cudaError_t reduce_t(int g, const uint8_t* const* c, const float* const* s, int64_t n, uint8_t* oc, float* os,
                     float* of, cudaStream_t st, const SyncArgs& sy) {
  using J = ReduceJob<BIN, GT, MODE, BOUT>;
  const TileGeo geo = pick([g](int te) { return J::in_bytes(te, g); }, [](int te) { return J::out_bytes(te); });
  J job{};
  for (int p = 0; p < g; ++p) {
    job.c[p] = c[p];
    job.s[p] = s[p];
  }
  job.g = g;
  job.n = n;
  job.oc = oc;
  job.os = os;
  job.of = of;
  job.te = geo.te;
  return launch_job(job, geo, (n + geo.te - 1) / geo.te, st, sy);
}

template <int BIN, int MODE, int BOUT>
cudaError_t reduce_g(int g, const uint8_t* const* c, const float* const* s, int64_t n, uint8_t* oc, float* os,
                     float* of, cudaStream_t st, const SyncArgs& sy) {
  switch (g) {
    case 1: return reduce_t<BIN, 1, MODE, BOUT>(g, c, s, n, oc, os, of, st, sy);
    case 2: return reduce_t<BIN, 2, MODE, BOUT>(g, c, s, n, oc, os, of, st, sy);
    case 4: return reduce_t<BIN, 4, MODE, BOUT>(g, c, s, n, oc, os, of, st, sy);
    case 8: return reduce_t<BIN, 8, MODE, BOUT>(g, c, s, n, oc, os, of, st, sy);
    default: return reduce_t<BIN, 0, MODE, BOUT>(g, c, s, n, oc, os, of, st, sy);
  }
}

}  // namespace

bool tiles_on() {
  static const bool on = tune_param("tma", 0) != 0;   // measured slower: off by default
  return on;
}

cudaError_t tiles_quantize(const void* x, hz_dtype dt, int64_t n, int bits, int block, uint8_t* codes, float* scales,
                           void* y, hz_dtype out_dt, int acc, cudaStream_t st, const SyncArgs& sy) {
  if (!tiles_on() || block != 256 || n <= 0 || n % 1024 != 0 || (y && acc) || (bits != 8 && bits != 4) ||
      !a16(x) || !a16(codes) || !a16(scales) || !a16(y) || (!codes && !y))
    return cudaErrorNotSupported;
  const int out = out_code(y != nullptr, out_dt);
  switch (dt) {
    case HZ_F32:
      return bits == 8 ? quant_o<float, 8>(x, n, codes, scales, y, out, st, sy)
                       : quant_o<float, 4>(x, n, codes, scales, y, out, st, sy);
    case HZ_BF16:
      return bits == 8 ? quant_o<__nv_bfloat16, 8>(x, n, codes, scales, y, out, st, sy)
                       : quant_o<__nv_bfloat16, 4>(x, n, codes, scales, y, out, st, sy);
    case HZ_F16:
      return bits == 8 ? quant_o<__half, 8>(x, n, codes, scales, y, out, st, sy)
                       : quant_o<__half, 4>(x, n, codes, scales, y, out, st, sy);
  }
  return cudaErrorNotSupported;
}

static bool pieces_ok(const Pieces& pc) {
  if (pc.n < 1 || pc.len <= 0 || pc.len % 1024 != 0) return false;
  for (int j = 0; j < pc.n; ++j)
    if (!a16(pc.c[j]) || !a16(pc.s[j])) return false;
  if (pc.sec_c) {
    if (!a16(pc.sec_c) || !a16(pc.sec_s) || pc.sec_lo % pc.len != 0 || pc.sec_hi % pc.len != 0) return false;
  }
  return true;
}

cudaError_t tiles_gather(const Pieces& pc, int bits, int block, void* y, hz_dtype out_dt, cudaStream_t st,
                         const SyncArgs& sy) {
  if (!tiles_on() || block != 256 || (bits != 8 && bits != 4) || !pieces_ok(pc) || !a16(y))
    return cudaErrorNotSupported;
  switch (out_dt) {
    case HZ_BF16: return bits == 8 ? gather_t<8, __nv_bfloat16>(pc, y, st, sy) : gather_t<4, __nv_bfloat16>(pc, y, st, sy);
    case HZ_F16: return bits == 8 ? gather_t<8, __half>(pc, y, st, sy) : gather_t<4, __half>(pc, y, st, sy);
    case HZ_F32: return bits == 8 ? gather_t<8, float>(pc, y, st, sy) : gather_t<4, float>(pc, y, st, sy);
  }
  return cudaErrorNotSupported;
}

cudaError_t tiles_dual(const Pieces& pc, void* y, const void* x, hz_dtype dt, int64_t nq, int qbits, uint8_t* codes,
                       float* scales, float* qy, int acc, cudaStream_t st, const SyncArgs& sy) {
  if (!tiles_on() || !pieces_ok(pc) || !a16(y) || !a16(x) || nq <= 0 || nq % 1024 != 0 || (qy && acc) ||
      (!qy && (!a16(codes) || !a16(scales) || !codes)) || !a16(qy))
    return cudaErrorNotSupported;
#define HZ_DUAL(T)                                                                                   \
  if (qy) return qbits == 8 ? dual_t<T, 8, 3>(pc, y, x, nq, nullptr, nullptr, qy, st, sy)             \
                            : dual_t<T, 4, 3>(pc, y, x, nq, nullptr, nullptr, qy, st, sy);            \
  return qbits == 8 ? dual_t<T, 8, 0>(pc, y, x, nq, codes, scales, nullptr, st, sy)                   \
                    : dual_t<T, 4, 0>(pc, y, x, nq, codes, scales, nullptr, st, sy);
  switch (dt) {
    case HZ_F32: { HZ_DUAL(float) }
    case HZ_BF16: { HZ_DUAL(__nv_bfloat16) }
    case HZ_F16: { HZ_DUAL(__half) }
  }
#undef HZ_DUAL
  return cudaErrorNotSupported;
}

cudaError_t tiles_reduce(int g, const uint8_t* const* c, const float* const* s, int64_t n, int bits_in, int block,
                         int bits_out, uint8_t* oc, float* os, float* of, int acc, cudaStream_t st,
                         const SyncArgs& sy) {
  if (!tiles_on() || block != 256 || n <= 0 || n % 1024 != 0 || g < 1 || g > kMaxG) return cudaErrorNotSupported;
  for (int p = 0; p < g; ++p)
    if (!a16(c[p]) || !a16(s[p])) return cudaErrorNotSupported;
  if (bits_out == 0) {
    if (!a16(of)) return cudaErrorNotSupported;
    if (acc) return bits_in == 8 ? reduce_g<8, 1, 0>(g, c, s, n, oc, os, of, st, sy)
                                 : reduce_g<4, 1, 0>(g, c, s, n, oc, os, of, st, sy);
    return bits_in == 8 ? reduce_g<8, 0, 0>(g, c, s, n, oc, os, of, st, sy)
                        : reduce_g<4, 0, 0>(g, c, s, n, oc, os, of, st, sy);
  }
  if (!a16(oc) || !a16(os)) return cudaErrorNotSupported;
  if (bits_in == 8) return bits_out == 8 ? reduce_g<8, 2, 8>(g, c, s, n, oc, os, of, st, sy)
                                         : reduce_g<8, 2, 4>(g, c, s, n, oc, os, of, st, sy);
  return bits_out == 8 ? reduce_g<4, 2, 8>(g, c, s, n, oc, os, of, st, sy)
                       : reduce_g<4, 2, 4>(g, c, s, n, oc, os, of, st, sy);
}

}  // namespace hz
