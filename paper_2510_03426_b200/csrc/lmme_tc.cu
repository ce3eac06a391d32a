// tcgen05 LMME for complex64 GOOMs: Eq. 10-12 with the real GEMM on the 5th-gen
// tensor cores at FP32 accuracy (3xTF32), everything else fused around it.
//
// One CTA = one 128 x BN output tile (BN = 256, or 128 when m % 256 != 0), full K.
// Warp roles, all synchronised by mbarriers:
//   warp 0      loader   : cp.async.bulk copies of the raw complex64 K-blocks
//                          (A: 128 rows x 16 k, B: 16 k x BN) into a RAW ring;
//   warp 1      MMA      : one thread issues, per 8-wide K step, three
//                          tcgen05.mma.cta_group::1.kind::tf32 into one FP32 TMEM
//                          accumulator: small*big + big*small + big*big;
//   warps 2..9  transform: RAW ring -> operand ring: v = sign * exp(log - scale)
//                          (clamped row / column scales from the pre-pass), split
//                          v = big + small (TF32, round-to-nearest), written into
//                          the 64B-swizzled K-major layout the UMMA descriptors
//                          read. No intermediate real matrix touches HBM.
//   warps 2..9  epilogue : tcgen05.ld the accumulator, (log|I| + a_i) + b_j and the
//                          sign in registers, optional fused gadd with D, store.
//
// Error budget: plain TF32 gives ~3e-4 Frobenius error at d = 1024;
// 3xTF32 with FP32 accumulation matches FP32 SIMT. The exponential is
// ex2.approx((log - scale) * log2 e) (rel. error ~2^-22 near the row maximum,
// where the products that matter live), non-FTZ so subnormals survive.
#include "goom_internal.cuh"

namespace goom {

namespace {

constexpr int BM = 128;
constexpr int BK = 16;  // K per stage: 16 TF32 = one 64-byte swizzle row
constexpr int RAW_STAGES = 2;
constexpr int OP_STAGES = 2;
constexpr int kXformWarps = 8;
constexpr int kXform = kXformWarps * 32;
constexpr int kThreads = 64 + kXform;  // loader warp, MMA warp, transform warps

template <int BN>
struct Cfg {
  static constexpr int kRawA = BM * BK * 8;       // complex64
  static constexpr int kRawB = BK * BN * 8;
  static constexpr int kRawStage = kRawA + kRawB;
  static constexpr int kOpA = BM * BK * 4;        // one TF32 plane
  static constexpr int kOpB = BN * BK * 4;
  static constexpr int kOpStage = 2 * kOpA + 2 * kOpB;
  static constexpr int kTmemCols = BN;
  static constexpr int kRingBytes = RAW_STAGES * kRawStage + OP_STAGES * kOpStage;
  static constexpr int kSmem = kRingBytes + 1024 + 256 + (BM + BN) * 4;
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
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
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
__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {  // non-FTZ: keeps subnormals
  float r;
  asm("ex2.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// K-major operand, 64B swizzle: rows of 64 B (16 TF32), 8-row atoms of 512 B.
__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | (1ull << 16) | ((uint64_t)(512 >> 4) << 32) |
         (1ull << 46) | (4ull << 61);
}
// byte offset of 16-byte chunk c (4 TF32 along K) of row r: Swizzle<2,4,3>
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
               "r"(d));
}

constexpr float kLog2e = 1.4426950408889634f;

// sign * exp(log - scale) split into TF32 (big, small). `canon` = every imaginary part of
// the chunk is exactly 0 or pi (our kernels always emit that); otherwise cos() decides.
__device__ __forceinline__ void goom_split(float2 z, float scale, bool canon, uint32_t& big,
                                           uint32_t& small) {
  // (log - scale) first: exact near the row maximum even for |log| ~ 1e6 (a pre-scaled
  // FFMA would round scale * log2 e at |scale| ulp and lose the whole mantissa)
  float e = ex2_approx(__fsub_rn(z.x, scale) * kLog2e);
  float v;
  if (canon) v = z.y != 0.0f ? -e : e;
  else v = goom_sign(z.y) * e;
  big = tf32_rna(v);
  small = tf32_rna(v - __uint_as_float(big));
}
__device__ __forceinline__ bool canonical(float y) { return y == 0.0f || y == kPi; }

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    lmme_tc_kernel(Operand A, Operand B, Operand D, Scales rowA, Scales colB,
                   float2* __restrict__ C, int64_t strideC, int64_t b_base, int n, int k, int m) {
  using G = Cfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* op_ring = smem;                               // OP_STAGES x kOpStage (1 KB aligned)
  uint8_t* raw_ring = smem + OP_STAGES * G::kOpStage;    // RAW_STAGES x kRawStage
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + G::kRingBytes);
  uint64_t* raw_full = bars;                     // [RAW_STAGES]
  uint64_t* raw_empty = bars + RAW_STAGES;       // [RAW_STAGES]
  uint64_t* op_full = bars + 2 * RAW_STAGES;     // [OP_STAGES]
  uint64_t* op_empty = op_full + OP_STAGES;      // [OP_STAGES]
  uint64_t* acc_done = op_empty + OP_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);
  float* sScaleA = reinterpret_cast<float*>(smem + G::kRingBytes + 256);
  float* sScaleB = sScaleA + BM;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t b = b_base + blockIdx.z;
  const int row0 = blockIdx.y * BM;
  const int col0 = blockIdx.x * BN;
  const int nk = k / BK;

  const float2* a = A.at(b);
  const float2* bm = B.at(b);
  const float* ra = rowA.at(b);
  const float* cb = colB.at(b);

  if (tid == 0) {
    for (int s = 0; s < RAW_STAGES; ++s) {
      mbar_init(smem_u32(&raw_full[s]), 1);
      mbar_init(smem_u32(&raw_empty[s]), kXform);
    }
    for (int s = 0; s < OP_STAGES; ++s) {
      mbar_init(smem_u32(&op_full[s]), kXform);
      mbar_init(smem_u32(&op_empty[s]), 1);
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

  if (warp == 0) {
    // ------------------------------ loader ------------------------------
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % RAW_STAGES;
      mbar_wait(smem_u32(&raw_empty[s]), ((kb / RAW_STAGES) & 1) ^ 1);
      const uint32_t full = smem_u32(&raw_full[s]);
      if (lane == 0) mbar_expect_tx(full, G::kRawStage);
      __syncwarp();
      const uint32_t dA = smem_u32(raw_ring + s * G::kRawStage);
      const uint32_t dB = dA + G::kRawA;
      const int k0 = kb * BK;
      for (int r = lane; r < BM; r += 32)  // 128 row segments of 128 B
        bulk_g2s(dA + r * (BK * 8), a + (int64_t)(row0 + r) * k + k0, BK * 8, full);
      if (lane < BK)  // 16 row segments of BN * 8 B
        bulk_g2s(dB + lane * (BN * 8), bm + (int64_t)(k0 + lane) * m + col0, BN * 8, full);
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ------------------------------
    if (lane == 0) {
      constexpr uint32_t idesc = tf32_idesc(BM, BN);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % OP_STAGES;
        mbar_wait(smem_u32(&op_full[s]), (kb / OP_STAGES) & 1);
        tc_fence_after();
        const uint32_t base = smem_u32(op_ring + s * G::kOpStage);
        const uint64_t dAb = sw64_desc(base), dAs = sw64_desc(base + G::kOpA);
        const uint64_t dBb = sw64_desc(base + 2 * G::kOpA);
        const uint64_t dBs = sw64_desc(base + 2 * G::kOpA + G::kOpB);
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint64_t adv = (uint64_t)(kk * 32) >> 4;  // 8 TF32 = 32 B along K
          mma_tf32(tmem, dAs + adv, dBb + adv, idesc, (kb | kk) != 0);
          mma_tf32(tmem, dAb + adv, dBs + adv, idesc, 1);
          mma_tf32(tmem, dAb + adv, dBb + adv, idesc, 1);
        }
        mma_commit(smem_u32(&op_empty[s]));  // frees the operand stage when these MMAs finish
      }
      mma_commit(smem_u32(acc_done));        // accumulator complete
    }
    __syncwarp();
  } else {
    // ------------------------------ transform ------------------------------
    const int t = tid - 64;
    for (int kb = 0; kb < nk; ++kb) {
      const int rs = kb % RAW_STAGES, os = kb % OP_STAGES;
      mbar_wait(smem_u32(&raw_full[rs]), (kb / RAW_STAGES) & 1);
      mbar_wait(smem_u32(&op_empty[os]), ((kb / OP_STAGES) & 1) ^ 1);
      const uint8_t* rawA = raw_ring + rs * G::kRawStage;
      const float2* rawB = reinterpret_cast<const float2*>(rawA + G::kRawA);
      const uint32_t base = smem_u32(op_ring + os * G::kOpStage);
      const uint32_t aBig = base, aSmall = base + G::kOpA;
      const uint32_t bBig = base + 2 * G::kOpA, bSmall = bBig + G::kOpB;
      // A: 128 rows x 4 chunks (4 k each) = 512 chunks
#pragma unroll
      for (int i = 0; i < (BM * 4) / kXform; ++i) {
        const int q = t + i * kXform;
        const int r = q >> 2, c = q & 3;
        const float4* src = reinterpret_cast<const float4*>(rawA + r * (BK * 8) + c * 32);
        const float4 p0 = src[0], p1 = src[1];
        const float sc = sScaleA[r];
        const bool canon = canonical(p0.y) && canonical(p0.w) && canonical(p1.y) && canonical(p1.w);
        uint32_t hb[4], lb[4];
        goom_split(make_float2(p0.x, p0.y), sc, canon, hb[0], lb[0]);
        goom_split(make_float2(p0.z, p0.w), sc, canon, hb[1], lb[1]);
        goom_split(make_float2(p1.x, p1.y), sc, canon, hb[2], lb[2]);
        goom_split(make_float2(p1.z, p1.w), sc, canon, hb[3], lb[3]);
        const uint32_t off = sw64_off(r, c);
        st_shared_v4(aBig + off, hb[0], hb[1], hb[2], hb[3]);
        st_shared_v4(aSmall + off, lb[0], lb[1], lb[2], lb[3]);
      }
      // B: BN columns (UMMA rows) x 4 chunks; lanes run along n (conflict-free reads)
#pragma unroll
      for (int i = 0; i < (BN * 4) / kXform; ++i) {
        const int q = t + i * kXform;
        const int nn = q % BN, c = q / BN;
        const float sc = sScaleB[nn];
        float2 z[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) z[j] = rawB[(4 * c + j) * BN + nn];
        const bool canon = canonical(z[0].y) && canonical(z[1].y) && canonical(z[2].y) &&
                           canonical(z[3].y);
        uint32_t hb[4], lb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) goom_split(z[j], sc, canon, hb[j], lb[j]);
        const uint32_t off = sw64_off(nn, c);
        st_shared_v4(bBig + off, hb[0], hb[1], hb[2], hb[3]);
        st_shared_v4(bSmall + off, lb[0], lb[1], lb[2], lb[3]);
      }
      mbar_arrive(smem_u32(&raw_empty[rs]));
      fence_async_smem();
      mbar_arrive(smem_u32(&op_full[os]));
    }

    // ------------------------------ epilogue ------------------------------
    mbar_wait(smem_u32(acc_done), 0);
    tc_fence_after();
    const int quad = warp & 3;            // TMEM lane quadrant this warp may access
    const int part = (warp - 2) >> 2;     // which half of the columns
    const int row = quad * 32 + lane;
    const float ai = sScaleA[row];
    float2* crow = C + b * strideC + (int64_t)(row0 + row) * m + col0;
    const float2* drow = D.ptr ? D.at(b) + (int64_t)(row0 + row) * m + col0 : nullptr;
#pragma unroll 1
    for (int chunk = 0; chunk < BN / 64; ++chunk) {
      const int col = part * (BN / 2) + chunk * 32;
      uint32_t v[32];
      tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)col, v);
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        float2 o0 = lmme_out<float>(__uint_as_float(v[j]), ai, sScaleB[col + j]);
        float2 o1 = lmme_out<float>(__uint_as_float(v[j + 1]), ai, sScaleB[col + j + 1]);
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

template <int BN>
int launch_tc(const LmmeProblem& p, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(lmme_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg<BN>::kSmem) != cudaSuccess)
      return cuda_fail(cudaGetLastError(), "lmme_tc smem attribute");
    attr_set = true;
  }
  const int64_t zmax = 65535;
  for (int64_t b0 = 0; b0 < p.batch; b0 += zmax) {
    int64_t nb = p.batch - b0 < zmax ? p.batch - b0 : zmax;
    dim3 grid(p.m / BN, p.n / BM, (unsigned)nb);
    lmme_tc_kernel<BN><<<grid, kThreads, Cfg<BN>::kSmem, s>>>(p.A, p.B, p.D, p.rowA, p.colB, p.C,
                                                              p.strideC, b0, p.n, p.k, p.m);
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
  // bulk copies need 16-byte aligned rows: every operand base / stride is a multiple of 16 B
  if ((reinterpret_cast<uintptr_t>(p.A.ptr) | reinterpret_cast<uintptr_t>(p.B.ptr)) & 15)
    return GOOM_EUNSUPPORTED;
  if (p.m % 256 == 0) return launch_tc<256>(p, s);
  return launch_tc<128>(p, s);
}

}  // namespace goom
