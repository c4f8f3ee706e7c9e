// The TMA tile engine: a codec kernel whose every byte moves by bulk copy (HZ_TUNE
// tma=1; OFF by default — measured slower than the LSU kernels, see below).  Internal header.
//
// Design: cp.async.bulk global -> shared into a ring of S input stages completed on
// mbarriers (peer pieces over NVLink the same way), the codec transform shared -> shared
// by all threads, cp.async.bulk shared -> global of the output from two output buffers.
// The in-flight bytes are held in shared memory by the copy engine instead of registers
// and L1.  Motivation: a plain streaming kernel with the codec's write-heavy byte mixes
// reaches 5.24-5.66 TB/s with ld/st.global and 5.59-6.02 TB/s with bulk copies
// (tools/tma_mix_probe.cu vs tools/hbm_mix_probe.cu, profiles/tma_r02.md).
// Measured in the product (profiles/tma_r02.md): the engine LOSES on every hot shape —
// N = 1 round trip 57-63 µs vs 51 µs, dequantize 29.5-33.6 vs 27.9 µs; N = 2 dual
// gather || quantize 86.7 vs 57.4 µs — because the codec's per-tile arithmetic (block
// absmax shuffles, two IEEE divisions per block, packing) sits between two CTA barriers
// per tile, serialised with the copies of its CTA, while the LSU kernels overlap the
// same arithmetic across 32 independent warps per SM.  It stays selectable, parity-
// tested (tests/test_gpu_tiles.py), as the reproducible evidence for that choice.
//
#pragma once

#include "codec.cuh"

namespace hz {
namespace dev {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
}
// bulk load global -> shared (bytes % 16 == 0, src / dst 16-byte aligned), completion
// counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

// bulk store shared -> global (bytes % 16 == 0, both 16-byte aligned), in the current
// bulk group
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// host-chosen pipeline geometry: te elements per tile (multiple of 1024), S input
// stages of ib bytes, 2 output buffers of ob bytes (all multiples of 128)
struct TileGeo {
  int te;
  int S;
  int ib;
  int ob;
  __host__ __device__ __forceinline__ int smem() const { return S * ib + 2 * ob + S * 8; }
};

struct Pipe {
  char* in;
  char* out;
  uint64_t* bar;
  int S, ib, ob;
  __device__ __forceinline__ char* inb(int64_t i) const { return in + (i % S) * ib; }
  __device__ __forceinline__ char* outb(int64_t i) const { return out + (i & 1) * ob; }
  __device__ __forceinline__ uint64_t* full(int64_t i) const { return bar + (i % S); }
  __device__ __forceinline__ unsigned parity(int64_t i) const { return static_cast<unsigned>((i / S) & 1); }
};

__device__ __forceinline__ Pipe pipe_init(char* smem, const TileGeo& g) {
  Pipe p{smem, smem + g.S * g.ib, reinterpret_cast<uint64_t*>(smem + g.S * g.ib + 2 * g.ob), g.S, g.ib, g.ob};
  if (threadIdx.x == 0) {
    for (int s = 0; s < g.S; ++s) mbar_init(p.bar + s, 1);
    mbar_init_fence();
  }
  __syncthreads();
  return p;
}

template <class Job>
__device__ __forceinline__ void run_tiles(const Job& job, const Pipe& p, int64_t first, int64_t stride) {
  const int64_t total = job.ntiles();
  const int64_t mine = total > first ? (total - first + stride - 1) / stride : 0;
  if (threadIdx.x == 0) {
    fence_proxy_async();
    for (int64_t i = 0; i < p.S && i < mine; ++i) job.load(first + i * stride, p.inb(i), p.full(i));
  }
  for (int64_t i = 0; i < mine; ++i) {
    const int64_t t = first + i * stride;
    mbar_wait(p.full(i), p.parity(i));
    if (threadIdx.x == 0) bulk_wait_read1();   // the stores of tile i - 2 have read out buffer i % 2
    __syncthreads();
    job.compute(t, p.inb(i), p.outb(i));
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      job.store(t, p.outb(i));
      bulk_commit();
      if (i + p.S < mine) {
        fence_proxy_async();
        job.load(first + (i + p.S) * stride, p.inb(i), p.full(i));
      }
    }
  }
  if (threadIdx.x == 0) {
    bulk_wait_all();
    fence_proxy_async();
  }
}

// ------------------------------------------------------------------ quantize job
// x (T) -> codes (BITS) + fp32 scales per 256-element block, and with OUT 1 / 2 / 3 the
// round trip x_hat = fl(code * scale) as bf16 / fp16 / fp32 (a level whose exchange
// group has one member; codes may then be nullptr: not stored).
template <int OUT>
struct OutT;
template <>
struct OutT<0> { using T = float; static constexpr int bytes = 0; };
template <>
struct OutT<1> { using T = __nv_bfloat16; static constexpr int bytes = 2; };
template <>
struct OutT<2> { using T = __half; static constexpr int bytes = 2; };
template <>
struct OutT<3> { using T = float; static constexpr int bytes = 4; };

template <typename T, int BITS, int OUT>
struct QuantJob {
  using TO = typename OutT<OUT>::T;
  const T* x;
  int64_t n;          // elements, multiple of 1024
  uint8_t* codes;     // nullptr: round trip only (no codes / scales in the out buffer)
  float* scales;
  TO* y;              // OUT > 0
  int te;
  // out buffer: y [te*|TO|] | codes [te*BITS/8] | scales [te/64]
  __device__ __forceinline__ int codes_off() const { return te * OutT<OUT>::bytes; }
  __device__ __forceinline__ int scales_off() const { return codes_off() + te * BITS / 8; }
  __device__ __forceinline__ int64_t ntiles() const { return (n + te - 1) / te; }
  __device__ __forceinline__ int cnt(int64_t t) const {
    const int64_t e0 = t * te;
    return n - e0 < te ? static_cast<int>(n - e0) : te;
  }
  __device__ __forceinline__ void load(int64_t t, char* in, uint64_t* bar) const {
    const unsigned b = static_cast<unsigned>(cnt(t)) * sizeof(T);
    mbar_expect_tx(bar, b);
    bulk_g2s(in, x + t * te, b, bar);
  }
  // QU consecutive blocks per warp pass (the scale / inv divisions of the QU blocks run
  // on QU lanes at once, quantize_store); c is a multiple of 1024 = 4 blocks
  template <int QU>
  __device__ __forceinline__ void blocks(const char* in, char* out, int c) const {
    const int lane = threadIdx.x & 31;
    uint8_t* oc = codes ? reinterpret_cast<uint8_t*>(out + codes_off()) : nullptr;
    float* os = reinterpret_cast<float*>(out + scales_off());
    EmitOut<TO> emit{reinterpret_cast<TO*>(out)};
    const T* xs = reinterpret_cast<const T*>(in);
    for (int b = (threadIdx.x >> 5) * QU; b < c / 256; b += kThreads / 32 * QU) {
      In8<T> r[QU];
#pragma unroll
      for (int u = 0; u < QU; ++u) r[u].load_shared(xs + (b + u) * 256 + lane * 8);
      float v[QU][1][8];
      float am[QU];
#pragma unroll
      for (int u = 0; u < QU; ++u) {
        r[u].get(v[u][0]);
        float m = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) m = fmaxf(m, fabsf(v[u][0][i]));
        am[u] = group_max<32>(m);
      }
      if constexpr (OUT == 0) quantize_store<256, BITS, QU, NoEmit>(v, am, b, lane, oc, os, NoEmit{});
      else quantize_store<256, BITS, QU, EmitOut<TO>>(v, am, b, lane, oc, os, emit);
    }
  }
  __device__ __forceinline__ void compute(int64_t t, const char* in, char* out) const {
    const int c = cnt(t);
    if (c == te && te % (kThreads / 32 * 4 * 256) == 0) blocks<4>(in, out, c);   // 4 blocks per warp pass
    else blocks<1>(in, out, c);
  }
  __device__ __forceinline__ void store(int64_t t, const char* out) const {
    const int c = cnt(t);
    const int64_t e0 = t * te;
    if constexpr (OUT > 0) bulk_s2g(y + e0, out, static_cast<unsigned>(c) * sizeof(TO));
    if (codes) {
      bulk_s2g(codes + e0 * BITS / 8, out + codes_off(), static_cast<unsigned>(c) * BITS / 8);
      bulk_s2g(scales + e0 / 256, out + scales_off(), static_cast<unsigned>(c) / 64);
    }
  }
  static constexpr int in_bytes(int te) { return te * static_cast<int>(sizeof(T)); }
  static constexpr int out_bytes(int te, bool has_codes) {
    return te * OutT<OUT>::bytes + (has_codes ? te * BITS / 8 + te / 64 : 0);
  }
};

// ------------------------------------------------------------------- gather job
// Gather+dequantize of pieces (codes of BITS, 256-element blocks) into y (TO): tiles lie
// inside one piece (tpp per piece).  Pieces may be peers' memory (the bulk loads read
// over NVLink).  With pc.sec_c the codes and scales of tiles inside [sec_lo, sec_hi) (a
// union of whole pieces) are also stored to the hpZ secondary.  Out buffer: y [te*|TO|] |
// codes [te*BITS/8] | scales [te/64].
template <int BITS, typename TO>
struct GatherJob {
  Pieces pc;
  TO* y;
  int te;
  int64_t tpp;   // tiles per piece
  __device__ __forceinline__ int64_t ntiles() const { return tpp * pc.n; }
  __device__ __forceinline__ void where(int64_t t, int& j, int64_t& e0, int& c) const {
    j = static_cast<int>(t / tpp);
    e0 = (t % tpp) * te;
    c = pc.len - e0 < te ? static_cast<int>(pc.len - e0) : te;
  }
  __device__ __forceinline__ void load(int64_t t, char* in, uint64_t* bar) const {
    int j, c;
    int64_t e0;
    where(t, j, e0, c);
    const unsigned cb = static_cast<unsigned>(c) * BITS / 8, sb = static_cast<unsigned>(c) / 64;
    mbar_expect_tx(bar, cb + sb);
    bulk_g2s(in, pc.c[j] + e0 * BITS / 8, cb, bar);
    bulk_g2s(in + te * BITS / 8, pc.s[j] + e0 / 256, sb, bar);
  }
  __device__ __forceinline__ bool in_sec(int64_t t) const {
    int j, c;
    int64_t e0;
    where(t, j, e0, c);
    const int64_t g0 = j * pc.len + e0;
    return pc.sec_c && g0 >= pc.sec_lo && g0 < pc.sec_hi;
  }
  __device__ __forceinline__ void compute(int64_t t, const char* in, char* out) const {
    int j, c;
    int64_t e0;
    where(t, j, e0, c);
    const float* sc = reinterpret_cast<const float*>(in + te * BITS / 8);
    TO* yo = reinterpret_cast<TO*>(out);
    for (int u = threadIdx.x; u < c / 8; u += kThreads) {
      Codes8<BITS> raw;
      raw.load_shared(in + u * BITS);
      const float s = sc[u >> 5];
      float cf[8], v[8];
      raw.decode(cf);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __fmul_rn(cf[k], s);
      Out8<TO>::store(yo + u * 8, v);
    }
    if (in_sec(t)) {   // secondary: the tile's codes and scales, copied to the out buffer
      const uint4* a = reinterpret_cast<const uint4*>(in);
      uint4* b = reinterpret_cast<uint4*>(out + te * static_cast<int>(sizeof(TO)));
      for (int k = threadIdx.x; k < c * BITS / 8 / 16; k += kThreads) b[k] = a[k];
      const int so = te * BITS / 8 / 16;   // scales region (16-byte units)
      for (int k = threadIdx.x; k < c / 64 / 16; k += kThreads) b[so + k] = a[so + k];
    }
  }
  __device__ __forceinline__ void store(int64_t t, const char* out) const {
    int j, c;
    int64_t e0;
    where(t, j, e0, c);
    const int64_t g0 = j * pc.len + e0;
    bulk_s2g(y + g0, out, static_cast<unsigned>(c) * sizeof(TO));
    if (in_sec(t)) {
      const char* sb = out + te * static_cast<int>(sizeof(TO));
      bulk_s2g(pc.sec_c + (g0 - pc.sec_lo) * BITS / 8, sb, static_cast<unsigned>(c) * BITS / 8);
      bulk_s2g(pc.sec_s + (g0 - pc.sec_lo) / 256, sb + te * BITS / 8, static_cast<unsigned>(c) / 64);
    }
  }
  static constexpr int in_bytes(int te) { return te * BITS / 8 + te / 64; }
  static constexpr int out_bytes(int te, bool has_sec) {
    return te * static_cast<int>(sizeof(TO)) + (has_sec ? te * BITS / 8 + te / 64 : 0);
  }
};

// --------------------------------------------------------------------- dual job
// The dual kernel's two independent jobs (gather of phase a || quantize of phase a + 1)
// as one tile space: gather and quantize tiles alternate while both last, so at any
// time about half the CTAs stream each job.
template <class GJ, class QJ>
struct DualJob {
  GJ g;
  QJ q;
  __device__ __forceinline__ int64_t ntiles() const { return g.ntiles() + q.ntiles(); }
  // -> (is_gather, tile of that job)
  __device__ __forceinline__ bool split(int64_t t, int64_t& u) const {
    const int64_t ng = g.ntiles(), nq = q.ntiles();
    const int64_t m = ng < nq ? ng : nq;
    if (t < 2 * m) {
      u = t >> 1;
      return (t & 1) == 0;
    }
    u = t - m;
    return ng > nq;
  }
  __device__ __forceinline__ void load(int64_t t, char* in, uint64_t* bar) const {
    int64_t u;
    if (split(t, u)) g.load(u, in, bar);
    else q.load(u, in, bar);
  }
  __device__ __forceinline__ void compute(int64_t t, const char* in, char* out) const {
    int64_t u;
    if (split(t, u)) g.compute(u, in, out);
    else q.compute(u, in, out);
  }
  __device__ __forceinline__ void store(int64_t t, const char* out) const {
    int64_t u;
    if (split(t, u)) g.store(u, out);
    else q.store(u, out);
  }
};

// ------------------------------------------------------------------- reduce job
// Level reduce (A9 / A10): g coded inputs -> acc = x_hat_0, acc = fl(acc + x_hat_p)
// ascending p, then MODE 0: fp32 out, 1: fp32 out += (old value loaded with the tile),
// 2: requantize to BOUT bits (block absmax, quantize_store).  In stage: codes of input p
// at p*te*BIN/8 | scales of p at g*te*BIN/8 + p*te/64 | (MODE 1) old fp32 [te].
template <int BIN, int GT, int MODE, int BOUT>
struct ReduceJob {
  const uint8_t* c[kMaxG];
  const float* s[kMaxG];
  int g;
  int64_t n;
  uint8_t* oc;
  float* os;
  float* of;
  int te;
  __device__ __forceinline__ int gg() const { return GT > 0 ? GT : g; }
  __device__ __forceinline__ int64_t ntiles() const { return (n + te - 1) / te; }
  __device__ __forceinline__ int cnt(int64_t t) const {
    const int64_t e0 = t * te;
    return n - e0 < te ? static_cast<int>(n - e0) : te;
  }
  __device__ __forceinline__ void load(int64_t t, char* in, uint64_t* bar) const {
    const int cn = cnt(t);
    const int64_t e0 = t * te;
    const int G = gg();
    const unsigned cb = static_cast<unsigned>(cn) * BIN / 8, sb = static_cast<unsigned>(cn) / 64;
    mbar_expect_tx(bar, G * (cb + sb) + (MODE == 1 ? static_cast<unsigned>(cn) * 4 : 0u));
    for (int p = 0; p < G; ++p) {
      bulk_g2s(in + p * (te * BIN / 8), c[p] + e0 * BIN / 8, cb, bar);
      bulk_g2s(in + G * (te * BIN / 8) + p * (te / 64), s[p] + e0 / 256, sb, bar);
    }
    if constexpr (MODE == 1) bulk_g2s(in + G * (te * BIN / 8 + te / 64), of + e0, static_cast<unsigned>(cn) * 4, bar);
  }
  __device__ __forceinline__ void compute(int64_t t, const char* in, char* out) const {
    const int cn = cnt(t);
    const int G = gg();
    const float* sc = reinterpret_cast<const float*>(in + G * (te * BIN / 8));
    if constexpr (MODE < 2) {
      const float4* old = reinterpret_cast<const float4*>(in + G * (te * BIN / 8 + te / 64));
      float4* o = reinterpret_cast<float4*>(out);
      for (int u = threadIdx.x; u < cn / 4; u += kThreads) {
        float acc[4];
        for (int p = 0; p < G; ++p) {
          Codes4<BIN> r;
          r.load_shared(in + p * (te * BIN / 8) + u * BIN / 2);
          const float sv = sc[p * (te / 256) + (u >> 6)];
          float cf[4];
          r.decode(cf);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float xh = __fmul_rn(cf[k], sv);
            acc[k] = p == 0 ? xh : __fadd_rn(acc[k], xh);
          }
        }
        float4 v = make_float4(acc[0], acc[1], acc[2], acc[3]);
        if constexpr (MODE == 1) {
          const float4 a = old[u];
          v.x = __fadd_rn(a.x, v.x);
          v.y = __fadd_rn(a.y, v.y);
          v.z = __fadd_rn(a.z, v.z);
          v.w = __fadd_rn(a.w, v.w);
        }
        o[u] = v;
      }
    } else {
      const int lane = threadIdx.x & 31;
      uint8_t* ocs = reinterpret_cast<uint8_t*>(out);
      float* oss = reinterpret_cast<float*>(out + te * BOUT / 8);
      constexpr int QU = 2;   // blocks per warp pass (cn is a multiple of 4 blocks)
      for (int b = (threadIdx.x >> 5) * QU; b < cn / 256; b += kThreads / 32 * QU) {
        float v[QU][1][8];
        for (int p = 0; p < G; ++p) {
#pragma unroll
          for (int u = 0; u < QU; ++u) {
            Codes8<BIN> r;
            r.load_shared(in + p * (te * BIN / 8) + ((b + u) * 256 + lane * 8) * BIN / 8);
            const float sv = sc[p * (te / 256) + b + u];
            float cf[8];
            r.decode(cf);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float xh = __fmul_rn(cf[k], sv);
              v[u][0][k] = p == 0 ? xh : __fadd_rn(v[u][0][k], xh);
            }
          }
        }
        float am[QU];
#pragma unroll
        for (int u = 0; u < QU; ++u) {
          float m = 0.f;
#pragma unroll
          for (int k = 0; k < 8; ++k) m = fmaxf(m, fabsf(v[u][0][k]));
          am[u] = group_max<32>(m);
        }
        quantize_store<256, BOUT, QU, NoEmit>(v, am, b, lane, ocs, oss, NoEmit{});
      }
    }
  }
  __device__ __forceinline__ void store(int64_t t, const char* out) const {
    const int cn = cnt(t);
    const int64_t e0 = t * te;
    if constexpr (MODE < 2) {
      bulk_s2g(of + e0, out, static_cast<unsigned>(cn) * 4);
    } else {
      bulk_s2g(oc + e0 * BOUT / 8, out, static_cast<unsigned>(cn) * BOUT / 8);
      bulk_s2g(os + e0 / 256, out + te * BOUT / 8, static_cast<unsigned>(cn) / 64);
    }
  }
  static constexpr int in_bytes(int te, int g) { return g * (te * BIN / 8 + te / 64) + (MODE == 1 ? te * 4 : 0); }
  static constexpr int out_bytes(int te) { return MODE < 2 ? te * 4 : te * BOUT / 8 + te / 64; }
};

}  // namespace dev
}  // namespace hz
