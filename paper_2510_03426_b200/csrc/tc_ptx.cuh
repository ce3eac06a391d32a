// PTX helpers shared by the tcgen05 LMME kernels (lmme_tc.cu: cta_group::1,
// lmme_tc2.cu: cta_group::2 CTA pairs): mbarriers, TMA, tcgen05 MMA / TMEM,
// the 3xTF32 operand split and the log epilogue, tensor-map encoding.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "goom_internal.cuh"

namespace goom {
namespace tc {

constexpr int kGroupBytes = 1024;  // 8 rows x 16 k complex64 == 2 x 512 B TF32 planes

// ---- PTX helpers ---------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
// suspend-hinted wait: the thread sleeps until the phase flips instead of spinning
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 0x989680;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared, completing on an mbarrier (transaction bytes)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
// L2 eviction-priority policies for the cache_hint forms below
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_3d_hint(uint32_t dst, const CUtensorMap* map, int c0,
                                                 int c1, int c2, uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_hint(uint32_t dst, const CUtensorMap* map, int c0,
                                                 int c1, int c2, int c3, uint32_t bar,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar),
      "l"(policy)
      : "memory");
}
// 16-byte global store with an L2 eviction policy (streamed outputs: evict_first)
__device__ __forceinline__ void st_global_v4_hint(void* p, float4 v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// round-to-nearest (ties away) to TF32 on the bit pattern; v is finite, |v| <= 1
__device__ __forceinline__ uint32_t tf32_round(float v) {
  return (__float_as_uint(v) + 0x1000u) & 0xFFFFE000u;
}

// K-major operand, 64B swizzle: rows of 64 B (16 TF32), 8-row atoms of 512 B, consecutive
// atoms 1 KB apart (the big and small planes of a group interleave).
__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | (1ull << 16) |
         ((uint64_t)(kGroupBytes >> 4) << 32) | (1ull << 46) | (4ull << 61);
}
// byte offset of 16-byte chunk c (4 TF32 along K) of row r (0..7) inside a 512 B atom
__device__ __forceinline__ uint32_t sw64_off(int r, int c) {
  return (uint32_t)(r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
}

__host__ __device__ constexpr uint32_t tf32_idesc(int M, int N) {
  return (1u << 4)                      // D: F32
         | (2u << 7) | (2u << 10)       // A, B: TF32
         | ((uint32_t)(N >> 3) << 17)   // N
         | ((uint32_t)(M >> 4) << 24);  // M ; A, B K-major (bits 15/16 = 0)
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
__device__ __forceinline__ float4 ld_shared_v4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ float2 ld_shared_v2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
  return v;
}

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.69314718055994531f;

// log|x| via MUFU.LG2 (non-FTZ: subnormal accumulators keep a finite log); log 0 = -inf
__device__ __forceinline__ float fast_log_abs(float x) {
  float r;
  asm("lg2.approx.f32 %0, %1;" : "=f"(r) : "f"(fabsf(x)));
  return r * kLn2;
}
__device__ __forceinline__ float2 tc_out(float acc, float a, float b) {
  return make_float2(__fadd_rn(__fadd_rn(fast_log_abs(acc), a), b), acc < 0.0f ? kPi : 0.0f);
}

// sign * exp(log - scale) split into TF32 (big, small); ~13 instructions, branch-free.
// (log - scale) first: exact near the row maximum even for |log| ~ 1e6 (a pre-scaled
// FFMA would round scale * log2 e at ulp(|scale|) and lose the mantissa). ex2 is FTZ:
// exponentials below 2^-126 of the scale flush (only a row lying entirely below
// e^-87 in the clamp regime notices; DESIGN.md numerics).
// kCanon: the pre-pass saw only phases 0 / pi, so "negative" is just imag != 0
// `small` is left in FP32: the tensor core reads it truncated to TF32 (error <= 2^-21 |v|,
// far below the FP32-accumulation floor measured in tools/precision_probe.py) — two
// instructions per element saved on the kernel's critical path.
template <bool kCanon>
__device__ __forceinline__ void goom_split(float2 z, float scale, uint32_t& big, uint32_t& small) {
  const float e = ex2_approx(__fsub_rn(z.x, scale) * kLog2e);
  const bool neg = kCanon ? (z.y != 0.0f) : phase_negative(z.y);
  const float v = neg ? -e : e;
  big = tf32_round(v);
  small = __float_as_uint(v - __uint_as_float(big));
}

// epilogue staging store: volatile (ordered with the other asm shared-memory accesses and
// the async-proxy fence that precedes a TMA store) but no "memory" clobber, so ordinary
// global loads (column scales, the fused bias) may be scheduled across it
__device__ __forceinline__ void st_shared_v4_staging(uint32_t addr, uint32_t a, uint32_t b,
                                                     uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d));
}
__device__ __forceinline__ void st_shared_v2(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}


inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

inline int encode_raw(CUtensorMap* map, const void* ptr, CUtensorMapDataType dt, int rank,
                      const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                      CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_NONE) {
  auto fn = encode_fn();
  if (!fn) return fail(GOOM_EUNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, dt, rank, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(GOOM_EUNSUPPORTED, "cuTensorMapEncodeTiled failed");
  return GOOM_OK;
}
// complex64 tensors move as int64 elements
inline int encode(CUtensorMap* map, const Operand& op, int rank, const cuuint64_t* dims,
                  const cuuint64_t* strides, const cuuint32_t* box,
                  CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_NONE) {
  return encode_raw(map, op.ptr, CU_TENSOR_MAP_DATA_TYPE_INT64, rank, dims, strides, box, swizzle);
}

// matrices addressed by an operand and their stride in elements
inline void mats_of(const Operand& op, int64_t batch, int rows, int cols, int64_t& mats,
                    int64_t& mstride) {
  mats = op.stride == 0 ? 1 : (batch - 1) / op.div + 1;
  mstride = op.stride == 0 ? (int64_t)rows * cols : op.stride;
}


// ---- CTA-pair (cluster of 2) helpers -------------------------------------------
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// arrive on the mbarrier at the same shared offset in CTA `rank` of this cluster. Default
// (.release.cta) semantics, as CUTLASS's ClusterBarrier::arrive: an explicit .release.cluster
// compiles to MEMBAR.ALL.GPU + ERRBAR per arrive (measured: the top stall of the first
// version of this kernel). The operand data itself is ordered for the tensor core by the
// writer's fence.proxy.async before the arrive.
__device__ __forceinline__ void mbar_arrive_rank(uint32_t bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"(rank));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void tma_load_5d_hint(uint32_t dst, const CUtensorMap* map, int c0,
                                                 int c1, int c2, int c3, int c4, uint32_t bar,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar),
      "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, int c4, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int c0, int c1,
                                             int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(src)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// TMA store with an L2 eviction policy (streamed outputs: evict_first)
__device__ __forceinline__ void tma_store_3d_hint(const CUtensorMap* map, uint32_t src, int c0,
                                                  int c1, int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint"
      " [%0, {%1, %2, %3}], [%4], %5;" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(src), "l"(policy)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// completion of every prior MMA of this thread -> arrive on the barrier at `bar` in BOTH CTAs
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}


// Fused-scale kernels (lmme_tc.cu, lmme_tc2.cu kFuse): the ring positions of one CTA (pair)
// in issue order. The first tile's scale stages, then per tile t the main K-blocks
// main(t, kb) with the NEXT tile's scale stages interleaved. Lateness lf (nk % lf == 0): the
// scale stages come lf per main stage in the last 1/lf of the tile (lf = 1: one per main
// stage; 2: "late", two per main stage in the second half), so the later the scale pass, the
// shorter a scale-read line waits in L2 for its main-pass re-read (and the denser the ring
// traffic at the end of a tile). Every role walks the same sequence, so slot and phase
// bookkeeping agree.
struct FuseSeq {
  int64_t t, step, tiles;
  int kb, nk, sub, skb;  // sub: 0 main, 1 .. lf scale stage skb of tile t + step
  int lf, h;             // h: the first main stage followed by scale stages (no per-step division)
  bool prologue;
  __device__ __forceinline__ FuseSeq(int64_t t0, int64_t step_, int64_t tiles_, int nk_,
                                     int lf_ = 1)
      : t(t0), step(step_), tiles(tiles_), kb(0), nk(nk_), sub(0), skb(0),
        lf(lf_ > 1 && nk_ % lf_ == 0 ? lf_ : 1), h(nk_ - nk_ / lf), prologue(true) {}
  __device__ __forceinline__ bool valid() const { return t < tiles; }
  __device__ __forceinline__ bool scale() const { return prologue || sub != 0; }
  // tile whose data the stage holds, and its K-block
  __device__ __forceinline__ int64_t tile() const { return sub ? t + step : t; }
  __device__ __forceinline__ int block() const { return prologue ? kb : (sub ? skb : kb); }
  __device__ __forceinline__ void next() {
    if (prologue) {
      if (++kb == nk) {
        prologue = false;
        kb = 0;
      }
      return;
    }
    if (t + step < tiles && kb >= h && sub < lf) {  // main(kb) -> scale(lf (kb - h) + i)
      ++sub;
      skb = lf * (kb - h) + sub - 1;
      return;
    }
    sub = 0;
    if (++kb == nk) {
      kb = 0;
      t += step;
    }
  }
};

// FuseSeq lateness for the pair kernel (GOOM_TC_LATE, default 8: d = 256 399 -> 390 us against
// 2, profiles/r2_fuse_lateness_ab.txt) and the one-SM kernel (GOOM_TC1_LATE, default 1), read
// once on the host
inline int fuse_lateness(const char* var, int dflt) {
  const char* e = getenv(var);
  const int v = e ? atoi(e) : dflt;
  return v >= 1 ? v : dflt;
}
// the lateness a launch with nk K-blocks per tile uses (host side, so the kernels' loops carry
// no extra work): at most half the tile's main stages carry scale stages (lf = nk, every scale
// stage after the last main stage, measured 8% slower at d = 256), and lf divides nk
inline int fit_lateness(int lf, int nk) {
  while (lf > 1 && (2 * lf > nk || nk % lf != 0)) lf >>= 1;
  return lf < 1 ? 1 : lf;
}

// per-slot phase bits of the shared ring (kFuse: slots carry main and scale stages)
template <int STAGES>
struct RingBits {
  int s = 0;
  uint32_t full = 0, mainp = 0, scalep = 0, last_scale = 0, used = 0;
  __device__ __forceinline__ uint32_t bit(uint32_t v) const { return (v >> s) & 1u; }
  __device__ __forceinline__ void advance(bool scale) {
    const uint32_t m = 1u << s;
    full ^= m;
    used |= m;
    if (scale) {
      scalep ^= m;
      last_scale |= m;
    } else {
      mainp ^= m;
      last_scale &= ~m;
    }
    s = s + 1 == STAGES ? 0 : s + 1;
  }
};

__device__ __forceinline__ bool odd_phase(float im) { return im != 0.0f && im != kPi; }

}  // namespace tc
}  // namespace goom
