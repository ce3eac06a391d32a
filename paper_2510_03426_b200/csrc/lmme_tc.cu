// tcgen05 LMME for complex64 GOOMs: Eq. 10-12 with the real GEMM on the 5th-gen
// tensor cores at FP32 accuracy (3xTF32), everything else fused around it.
//
// One CTA = one 128 x BN output tile (BN = 256, or 128 when m % 256 != 0), full K.
// A STAGES-deep ring of K-blocks (16 wide), each stage used twice in place:
//   warp 0      loader   : TMA (cp.async.bulk.tensor) of the raw complex64 K-block:
//                          A as 16 groups of 8 rows x 16 k, B as BN/8 groups of
//                          16 k x 8 columns; every group is 1 KB of complex64;
//   warps 2..17 transform: each warp owns whole groups; it reads a group into
//                          registers, v = sign * exp(log - scale) (clamped scales from
//                          the pre-pass), splits v = big + small (TF32, round to
//                          nearest) and writes the two 512 B TF32 planes of the group
//                          back into the SAME 1 KB, in the 64B-swizzled K-major
//                          layout the UMMA descriptors read (SBO = 1 KB, big and
//                          small planes interleaved per group). No real matrix ever
//                          touches HBM and no second ring is needed;
//   warp 1      MMA      : one thread issues per 8-wide K step three
//                          tcgen05.mma.cta_group::1.kind::tf32 into one FP32 TMEM
//                          accumulator: small*big + big*small + big*big;
//   warps 2..17 epilogue : tcgen05.ld the accumulator, (log|I| + a_i) + b_j and the
//                          sign in registers (log via lg2.approx: abs. error ~1e-7,
//                          below the FP32 ulp of the output), optional fused gadd, store.
//
// Error budget: plain TF32 gives ~3e-4 Frobenius error at d = 1024;
// 3xTF32 keeps the single-LMME Frobenius error below 1e-5 up to k = 1024 (the
// tensor core's FP32 accumulation, not the split, sets the floor; measured
// in tools/precision_probe.py).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "goom_internal.cuh"

namespace goom {

namespace {

constexpr int BM = 128;
constexpr int BK = 16;        // K per stage: 16 TF32 = one 64-byte swizzle row
constexpr int STAGES = 4;
constexpr int kXformWarps = 16;
constexpr int kThreads = 64 + kXformWarps * 32;  // loader warp, MMA warp, transform warps
constexpr int kGroupBytes = 1024;                // 8 rows x 16 k complex64 == 2 x 512 B TF32

template <int BN>
struct Cfg {
  static constexpr int kGroupsA = BM / 8;
  static constexpr int kGroupsB = BN / 8;
  static constexpr int kBytesA = kGroupsA * kGroupBytes;
  static constexpr int kStage = (kGroupsA + kGroupsB) * kGroupBytes;
  static constexpr int kTmemCols = BN;
  static constexpr int kRing = STAGES * kStage;
  static constexpr int kSmem = kRing + 1024 + 256 + (BM + BN) * 4;
};

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
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
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
template <bool kCanon>
__device__ __forceinline__ void goom_split(float2 z, float scale, uint32_t& big, uint32_t& small) {
  const float e = ex2_approx(__fsub_rn(z.x, scale) * kLog2e);
  const bool neg = kCanon ? (z.y != 0.0f) : phase_negative(z.y);
  const float v = neg ? -e : e;
  big = tf32_round(v);
  small = tf32_round(v - __uint_as_float(big));
}

__device__ __forceinline__ void st_shared_v2(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}

// Transform one stage in place (see the header comment). A group g: raw [8 rows][16 k];
// lane l reads 16 B (k-pair) at l*16 and 512 + l*16 -> rows l/8 and 4 + l/8, k-pair l%8,
// conflict-free; it writes its 2 TF32 of each row as 8-byte halves of the swizzled chunk.
// B group: raw [16 k][8 cols]; lane (n = l%8, c = l/8) gathers k = 4c..4c+3 of column n.
template <int NA, int NB, bool kCanon>
__device__ __forceinline__ void transform_stage(uint32_t base, int xw, int lane,
                                                const float* sScaleA, const float* sScaleB) {
#pragma unroll
  for (int g = xw; g < NA; g += kXformWarps) {
    const uint32_t grp = base + g * kGroupBytes;
    const int r = lane >> 3, kp = lane & 7;
    const float4 q0 = ld_shared_v4(grp + lane * 16);        // row r,   k = 2kp, 2kp+1
    const float4 q1 = ld_shared_v4(grp + 512 + lane * 16);  // row r+4
    uint32_t h0, l0, h1, l1, h2, l2, h3, l3;
    const float s0 = sScaleA[g * 8 + r], s1 = sScaleA[g * 8 + r + 4];
    goom_split<kCanon>(make_float2(q0.x, q0.y), s0, h0, l0);
    goom_split<kCanon>(make_float2(q0.z, q0.w), s0, h1, l1);
    goom_split<kCanon>(make_float2(q1.x, q1.y), s1, h2, l2);
    goom_split<kCanon>(make_float2(q1.z, q1.w), s1, h3, l3);
    const uint32_t o0 = sw64_off(r, kp >> 1) + (kp & 1) * 8;
    const uint32_t o1 = sw64_off(r + 4, kp >> 1) + (kp & 1) * 8;
    __syncwarp();  // the whole group is in registers before it is overwritten
    st_shared_v2(grp + o0, h0, h1);
    st_shared_v2(grp + 512 + o0, l0, l1);
    st_shared_v2(grp + o1, h2, h3);
    st_shared_v2(grp + 512 + o1, l2, l3);
  }
  const int bn = lane & 7, bc = lane >> 3;
#pragma unroll
  for (int gb = xw; gb < NB; gb += kXformWarps) {
    const uint32_t grp = base + (NA + gb) * kGroupBytes;
    const float sc = sScaleB[gb * 8 + bn];
    uint32_t hb[4], lb[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 z = ld_shared_v2(grp + (4 * bc + j) * 64 + bn * 8);
      goom_split<kCanon>(z, sc, hb[j], lb[j]);
    }
    const uint32_t off = sw64_off(bn, bc);
    __syncwarp();
    st_shared_v4(grp + off, hb[0], hb[1], hb[2], hb[3]);
    st_shared_v4(grp + 512 + off, lb[0], lb[1], lb[2], lb[3]);
  }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    lmme_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   Operand A, Operand B, Operand D, Scales rowA, Scales colB,
                   float2* __restrict__ C, int64_t strideC, int64_t b_base, int n, int k, int m,
                   const int* __restrict__ noncanon, int debug) {
  using G = Cfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KB-align the ring while keeping the pointer's shared-space provenance
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + G::kRing);
  uint64_t* full = bars;                 // [STAGES] TMA landed (tx bytes)
  uint64_t* ready = bars + STAGES;       // [STAGES] operands transformed (8 warp arrivals)
  uint64_t* freed = bars + 2 * STAGES;   // [STAGES] MMAs of the stage retired (commit)
  uint64_t* acc_done = bars + 3 * STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);
  float* sScaleA = reinterpret_cast<float*>(smem + G::kRing + 256);
  float* sScaleB = sScaleA + BM;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t b = b_base + blockIdx.z;
  const int row0 = blockIdx.y * BM;
  const int col0 = blockIdx.x * BN;
  const int nk = k / BK;
  const float* ra = rowA.at(b);
  const float* cb = colB.at(b);

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&ready[s]), kXformWarps);
      mbar_init(smem_u32(&freed[s]), 1);
    }
    mbar_init(smem_u32(acc_done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // the MMA warp owns the TMEM allocation
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(G::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid; i < BM; i += kThreads) sScaleA[i] = ra[row0 + i];
  for (int i = tid; i < BN; i += kThreads) sScaleB[i] = cb[col0 + i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t ring = smem_u32(smem);

  if (warp == 0) {
    // ------------------------------ loader ------------------------------
    if (lane == 0) {
      const int ma = A.stride == 0 ? 0 : (int)(b / A.div);
      const int mb = B.stride == 0 ? 0 : (int)(b / B.div);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(smem_u32(&freed[s]), ((kb / STAGES) & 1) ^ 1);
        const uint32_t bar = smem_u32(&full[s]);
        if (debug >= 3) {  // profiling aid: no loads
          mbar_arrive(bar);
          continue;
        }
        mbar_expect_tx(bar, G::kStage);
        const uint32_t dst = ring + s * G::kStage;
        const int k0 = kb * BK;
        tma_load_3d(dst, &mapA, k0, row0, ma, bar);                      // [128 rows][16 k]
        tma_load_4d(dst + G::kBytesA, &mapB, 0, k0, col0 / 8, mb, bar);  // [BN/8][16 k][8 cols]
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ------------------------------
    if (lane == 0) {
      constexpr uint32_t idesc = tf32_idesc(BM, BN);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(smem_u32(&ready[s]), (kb / STAGES) & 1);
        tc_fence_after();
        if (debug == 2) {  // profiling aid: skip the MMAs
          mma_commit(smem_u32(&freed[s]));
          continue;
        }
        const uint32_t base = ring + s * G::kStage;
        const uint64_t dAb = sw64_desc(base), dAs = sw64_desc(base + 512);
        const uint64_t dBb = sw64_desc(base + G::kBytesA), dBs = sw64_desc(base + G::kBytesA + 512);
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint64_t adv = (uint64_t)(kk * 32) >> 4;  // 8 TF32 = 32 B along K
          mma_tf32(tmem, dAs + adv, dBb + adv, idesc, (kb | kk) != 0);
          mma_tf32(tmem, dAb + adv, dBs + adv, idesc, 1);
          mma_tf32(tmem, dAb + adv, dBb + adv, idesc, 1);
        }
        mma_commit(smem_u32(&freed[s]));  // the stage returns to the loader when these retire
      }
      mma_commit(smem_u32(acc_done));
    }
    __syncwarp();
  } else {
    // ------------------------------ transform (in place) ------------------------------
    const int xw = warp - 2;
    const bool canon = noncanon != nullptr && *noncanon == 0;
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(smem_u32(&full[s]), (kb / STAGES) & 1);
      const uint32_t base = ring + s * G::kStage;
      if (debug != 1 && debug != 3) {
        if (canon)
          transform_stage<G::kGroupsA, G::kGroupsB, true>(base, xw, lane, sScaleA, sScaleB);
        else
          transform_stage<G::kGroupsA, G::kGroupsB, false>(base, xw, lane, sScaleA, sScaleB);
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&ready[s]));
    }

    // ------------------------------ epilogue ------------------------------
    mbar_wait(smem_u32(acc_done), 0);
    tc_fence_after();
    const int quad = warp & 3;            // TMEM lane quadrant this warp may access
    const int part = (warp - 2) >> 2;     // which quarter of the columns
    const int row = quad * 32 + lane;
    const float ai = sScaleA[row];
    float2* crow = C + b * strideC + (int64_t)(row0 + row) * m + col0;
    const float2* drow = D.ptr ? D.at(b) + (int64_t)(row0 + row) * m + col0 : nullptr;
#pragma unroll 1
    for (int chunk = 0; chunk < BN / 128; ++chunk) {
      const int col = part * (BN / 4) + chunk * 32;
      uint32_t v[32];
      tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)col, v);
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        float2 o0 = tc_out(__uint_as_float(v[j]), ai, sScaleB[col + j]);
        float2 o1 = tc_out(__uint_as_float(v[j + 1]), ai, sScaleB[col + j + 1]);
        if (drow) {
          o0 = gadd_elem(o0, drow[col + j]);
          o1 = gadd_elem(o1, drow[col + j + 1]);
        }
        *reinterpret_cast<float4*>(crow + col + j) = make_float4(o0.x, o0.y, o1.x, o1.y);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(G::kTmemCols));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

int encode(CUtensorMap* map, const Operand& op, int rank, const cuuint64_t* dims,
           const cuuint64_t* strides, const cuuint32_t* box) {
  auto fn = encode_fn();
  if (!fn) return fail(GOOM_EUNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_INT64, rank, const_cast<float2*>(op.ptr), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(GOOM_EUNSUPPORTED, "cuTensorMapEncodeTiled failed");
  return GOOM_OK;
}

// matrices addressed by an operand and their stride in elements
inline void mats_of(const Operand& op, int64_t batch, int rows, int cols, int64_t& mats,
                    int64_t& mstride) {
  mats = op.stride == 0 ? 1 : (batch - 1) / op.div + 1;
  mstride = op.stride == 0 ? (int64_t)rows * cols : op.stride;
}

// GOOM_TC_DEBUG (profiling only; results invalid): 1 skips the transform, 2 the MMAs,
// 3 the TMA loads and the transform, 4 the TMA loads
int tc_debug() {
  static int v = [] {
    const char* e = getenv("GOOM_TC_DEBUG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <int BN>
int launch_tc(const LmmeProblem& p, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(lmme_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg<BN>::kSmem) != cudaSuccess)
      return cuda_fail(cudaGetLastError(), "lmme_tc smem attribute");
    attr_set = true;
  }
  alignas(64) CUtensorMap mapA, mapB;
  int64_t mats, mstride;
  // A: (k, n, matrix) complex64 moved as int64, box 16 k x 128 rows
  mats_of(p.A, p.batch, p.n, p.k, mats, mstride);
  {
    cuuint64_t dims[3] = {(cuuint64_t)p.k, (cuuint64_t)p.n, (cuuint64_t)mats};
    cuuint64_t strides[2] = {(cuuint64_t)p.k * 8, (cuuint64_t)mstride * 8};
    cuuint32_t box[3] = {BK, BM, 1};
    GOOM_TRY(encode(&mapA, p.A, 3, dims, strides, box));
  }
  // B: (8 cols, k, m/8 column groups, matrix), box 8 x 16 k x BN/8 -> [group][k][8] in smem
  mats_of(p.B, p.batch, p.k, p.m, mats, mstride);
  {
    cuuint64_t dims[4] = {8, (cuuint64_t)p.k, (cuuint64_t)(p.m / 8), (cuuint64_t)mats};
    cuuint64_t strides[3] = {(cuuint64_t)p.m * 8, 64, (cuuint64_t)mstride * 8};
    cuuint32_t box[4] = {8, BK, BN / 8, 1};
    GOOM_TRY(encode(&mapB, p.B, 4, dims, strides, box));
  }
  const int64_t zmax = 65535;
  for (int64_t b0 = 0; b0 < p.batch; b0 += zmax) {
    int64_t nb = p.batch - b0 < zmax ? p.batch - b0 : zmax;
    dim3 grid(p.m / BN, p.n / BM, (unsigned)nb);
    lmme_tc_kernel<BN><<<grid, kThreads, Cfg<BN>::kSmem, s>>>(
        mapA, mapB, p.A, p.B, p.D, p.rowA, p.colB, p.C, p.strideC, b0, p.n, p.k, p.m, p.noncanon, tc_debug());
    GOOM_CHECK_LAUNCH("lmme_tc_kernel");
  }
  return GOOM_OK;
}

}  // namespace

bool lmme_tc_eligible(int n, int k, int m) {
  return n > 0 && k > 0 && m > 0 && n % BM == 0 && m % 128 == 0 && k % BK == 0;
}

int lmme_tc(const LmmeProblem& p, cudaStream_t s) {
  if (!lmme_tc_eligible(p.n, p.k, p.m)) return GOOM_EUNSUPPORTED;
  // TMA: 16-byte aligned bases and matrix strides
  if (((reinterpret_cast<uintptr_t>(p.A.ptr) | reinterpret_cast<uintptr_t>(p.B.ptr)) & 15) ||
      ((p.A.stride | p.B.stride) & 1))
    return GOOM_EUNSUPPORTED;
  if (p.m % 256 == 0) return launch_tc<256>(p, s);
  return launch_tc<128>(p, s);
}

}  // namespace goom
