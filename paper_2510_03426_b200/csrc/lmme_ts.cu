// Tile-scaled LMME on CTA pairs: the chain engine's combine for d a multiple of 256.
//
// Same product as Eq. 10-12 (core.py:242-261), with the operands kept between scan
// phases as tile-scaled fp32 (goom_internal.cuh: X_ij = U_ij exp(q[i][j/256]), G[J] =
// max_i q[i][J]) instead of complex64 logs. Why (measured, lmme_tc2.cu stage probes on
// B200): with complex64 operands the pair kernel moves 8 B per operand element through
// TMA, LDS and STS and spends an ex2 per element in the transform and an lg2 per output
// element in the epilogue; the load path alone takes as long as the MMAs. Here
//   * operands are 4 B/element: half the L2->SMEM and LDS bytes;
//   * the transform is one FMUL per element by a per-(row, block) factor exp(q - rowmax q)
//     (left operand) or a per-row factor exp(q - G) (right operand), then the 3xTF32 split;
//   * the epilogue writes U = S * 2^-e (exact power-of-two row normalisation of the
//     accumulator S within its 256-column block) and q = rowmax_A + G_B + e ln 2: no log;
//   * or, for prefixes that are only digested, it reduces (max log, log Frobenius,
//     finiteness) per 32 rows and never writes the product.
// Scales follow Eq. 11's clamp (core.py:252-253): a = max(row scale, 0), b = max(G, 0), so a
// shrinking chain underflows where the reference's float32 run does (GOOM_TS_SCALES=truemax
// opts out). They differ from the reference's per-COLUMN maxima of the right operand in one
// way that the format cannot avoid: an entry more than ~e^87 below the largest entry of its
// (row, 256-column block) — or a right-operand row whose block lies e^87 below the block's
// G — flushes. The public scan therefore runs the complex64 kernels (exact Eq. 11 per
// column) unless GOOM_CHAIN_TS=1; this engine serves the long-chain harness (config 3).
//
// Pipeline per CTA (pair tile 256 x 256, full K, cta_group::2 like lmme_tc2.cu):
//   warp 0       TMA: raw fp32 K-block (A [128 rows][16 k], B [16 k][128 cols]) into a
//                4-deep raw ring;
//   warps 2..17  transform raw -> (big, small) TF32 planes (64B-swizzled, K-major) in a
//                4-deep plane ring; arrive on the leader's plane_ready;
//   warp 1       (leader) 6 x tcgen05.mma.cta_group::2.kind::tf32 (M=N=256, K=8) per
//                K-block into a double-buffered TMEM accumulator;
//   warps 18..21 epilogue (GOOM complex64 | tile-scaled fp32 | digest partials).
#include <cstdlib>
#include <string>

#include "tc_ptx.cuh"

namespace goom {

namespace {
using namespace tc;

constexpr int kRowsCta = 128;
constexpr int kPairN = 256;
constexpr int BK = 16;
constexpr int kXformWarps = 16;
constexpr int kEpiWarps = 4;
constexpr int kThreads = 64 + (kXformWarps + kEpiWarps) * 32;  // 704
// One ring of stages, operands landed by TMA directly in the UMMA layouts and turned into
// (big, small) TF32 planes IN PLACE (big overwrites the raw value, small goes to its twin):
//   [A big 8 KB | A small 8 KB]  K-major, 64B swizzle: 16 atoms of 8 rows x 64 B (SBO 512)
//   [B big 8 KB | B small 8 KB]  MN-major, 128B swizzle: 4 column chunks of 32 (LBO 2 KB) x
//                                2 atoms of 8 k-rows x 128 B (SBO 1 KB)
// so there is no separate raw ring and every transform LDS/STS is a contiguous 512 B per warp.
constexpr int kHalf = 8192;
constexpr int kStage = 4 * kHalf;                              // 32 KB
constexpr int kOffAs = kHalf, kOffBb = 2 * kHalf, kOffBs = 3 * kHalf;
constexpr int kOutStage = 4096;                                // 32 rows x 128 B
constexpr int kMaxK = 1024;
// shared memory: ring (S x 32 KB) | output staging (32 KB, not used by the digest epilogue) |
// per-tile right-operand row factors (2 x kMaxK floats) | barriers
template <int kOut, int S>
struct Lay {
  // staging buffers per epilogue warp: 2 (a TMA store in flight while the next is written),
  // 1 when a 6-deep ring leaves no room for two
  static constexpr int kOutBufs = kOut == kTsOutDigest ? 0 : (S >= 6 ? 1 : 2);
  static constexpr int kOutBytes = kEpiWarps * kOutBufs * kOutStage;
  static constexpr int kOutOff = S * kStage;
  static constexpr int kFacOff = kOutOff + kOutBytes;
  static constexpr int kBarOff = kFacOff + 2 * kMaxK * 4;
  static constexpr int kSmem = kBarOff + 512 + 1024;
  static_assert(kSmem <= 232448, "shared memory budget");
};
constexpr int kTmemCols = 2 * kPairN;

// K-major 64B-swizzled operand: 8-row atoms 512 B apart
__device__ __forceinline__ uint64_t kmaj_sw64(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | (1ull << 16) | ((uint64_t)(512 >> 4) << 32) |
         (1ull << 46) | (4ull << 61);
}
// MN-major TF32 operand in the 128B_BASE32B layout (the only MN-major smem layout tcgen05
// accepts for 32-bit types; CUTLASS sm100_common.inl): 128 B rows along N, 32-byte chunks
// swizzled with the row index mod 4, 4-row atoms SBO = 512 B apart along K, 32-column chunks
// LBO = 2 KB apart along N. TMA lands it with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.
__device__ __forceinline__ uint64_t mnmaj_sw128_32b(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(2048 >> 4) << 16) |
         ((uint64_t)(512 >> 4) << 32) | (1ull << 46) | (1ull << 61);
}

template <int N>
struct Ring {
  int s = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next() {
    if (++s == N) {
      s = 0;
      ph ^= 1u;
    }
  }
};

// exp(q - ref) for q <= ref; exact zero for an all-zero row / block (q = -inf)
__device__ __forceinline__ float scale_factor(float q, float ref) {
  return q == kNegInf ? 0.0f : ex2_approx(__fsub_rn(q, ref) * kLog2e);
}
__device__ __forceinline__ float decode_g(uint32_t g) {
  return g == 0u ? kNegInf : ordered_to_float(g);
}

// v -> (big, small) TF32 bit patterns: big = RN-to-TF32(v), small = v - big (exact in FP32;
// the tensor core reads it truncated to TF32)
__device__ __forceinline__ void split_tf32(float v, uint32_t& big, uint32_t& small) {
  big = tf32_round(v);
  small = __float_as_uint(v - __uint_as_float(big));
}


struct PairGrid {
  int nct, nrt;
  int64_t tiles;
  __device__ __forceinline__ void at(int64_t t, int64_t& b, int& prow0, int& pcol0) const {
    const int ct = (int)(t % nct);
    const int64_t q = t / nct;
    prow0 = (int)(q % nrt) * 256;
    pcol0 = ct * kPairN;
    b = q / nrt;
  }
};

// chained phase 1 (TsProblem::chain_s): tile t is step t / tps + 1 of the block chains
struct ChainArgs {
  uint32_t* done;
  int s;
  int64_t tps;
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int kOut, int S, bool kChain>
__global__ void __launch_bounds__(kThreads, 1)
    lmme_ts_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ CUtensorMap mapOut, TsIn A, TsIn B, TsOut T,
                   float4* __restrict__ parts, PairGrid grid, int n, int k, int m, int debug,
                   ChainArgs ch, int clampz, int pdl) {
  using Y = Lay<kOut, S>;
  constexpr int kStages = S, kOutOff = Y::kOutOff;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Y::kBarOff);
  uint64_t* full = bars;                            // [S] local, TMA tx
  uint64_t* ready = full + kStages;                 // [S] leader, 32 transform warps
  uint64_t* freed = ready + kStages;                // [S] local, MMA commit (multicast)
  uint64_t* acc_full = freed + kStages;             // [2] local, MMA commit (multicast)
  uint64_t* acc_empty = acc_full + 2;               // [2] leader, 8 epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cta_rank();
  const int64_t cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int nk = k / BK;
  const int nJk = k / 256, nJm = m / 256;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&ready[s]), 2 * kXformWarps);
      mbar_init(smem_u32(&freed[s]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&acc_full[i]), 1);
      mbar_init(smem_u32(&acc_empty[i]), 2 * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (pdl) {
    // programmatic dependent launch: the next launch's CTAs may start their prologue
    // (barriers, TMEM, descriptor prefetch) as this grid's CTAs retire; nothing below reads
    // global memory before the previous grid has completed and flushed
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  const uint32_t tmem = *tmem_slot;
  const uint32_t base = smem_u32(smem);
  // tile -> (matrix pair b, row / column offsets, chain step); matrix indices of the
  // operands and the output: b / div (plain batch) or b s + step (chained phase 1)
  auto decode = [&](int64_t t, int64_t& b, int& prow0, int& pcol0, int& step) {
    if constexpr (kChain) {
      step = (int)(t / ch.tps) + 1;
      grid.at(t % ch.tps, b, prow0, pcol0);
    } else {
      step = 0;
      grid.at(t, b, prow0, pcol0);
    }
  };
  auto idx_a = [&](int64_t b, int step) -> int64_t {
    if constexpr (kChain) return b * ch.s + step;
    return A.sU == 0 ? 0 : b / A.div;
  };
  auto idx_b = [&](int64_t b, int step) -> int64_t {
    if constexpr (kChain) return b * ch.s + step - 1;
    return B.sU == 0 ? 0 : b / B.div;
  };
  auto idx_o = [&](int64_t b, int step) -> int64_t {
    if constexpr (kChain) return b * ch.s + step;
    return b;
  };
  // a chained step reads the previous step's output: column tile JB of block b is complete
  // once all (n / 256) row pairs x 2 CTAs of every earlier step have signalled
  // (warp-collective: lane 0 acquires, __syncwarp orders the other lanes' loads after it)
  auto dep_ready = [&](int64_t b, int JB, int step) -> bool {
    if (!kChain || step < 2) return true;
    int ok = 0;
    if (lane == 0)
      ok = ld_acquire_u32(ch.done + b * nJm + JB) >= (uint32_t)(2 * (n / 256) * (step - 1));
    ok = __shfl_sync(0xffffffffu, ok, 0);
    __syncwarp();
    return ok != 0;
  };
  auto dep_wait = [&](int64_t b, int JB, int step) {
    while (!dep_ready(b, JB, step)) __nanosleep(64);
  };

  if (warp == 0) {
    // ------------------------------ TMA loader ------------------------------
    if (lane == 0) {
      Ring<kStages> rr;
      for (int64_t t = cluster; t < grid.tiles; t += nclusters) {
        int64_t b;
        int prow0, pcol0, step;
        decode(t, b, prow0, pcol0, step);
        const int row0 = prow0 + (int)rank * kRowsCta;
        const int col0 = pcol0 + (int)rank * (kPairN / 2);
        const int ma = (int)idx_a(b, step);
        const int mb = (int)idx_b(b, step);
        if (kChain && step >= 2) {
          const uint32_t need = (uint32_t)(2 * (n / 256) * (step - 1));
          while (ld_acquire_u32(ch.done + b * nJm + pcol0 / 256) < need) __nanosleep(64);
          asm volatile("fence.proxy.async.global;" ::: "memory");  // acquire before TMA reads
        }
        for (int kb = 0; kb < nk; ++kb, rr.next()) {
          mbar_wait(smem_u32(&freed[rr.s]), rr.ph ^ 1u);
          const uint32_t bar = smem_u32(&full[rr.s]);
          mbar_expect_tx(bar, 2 * kHalf);
          const uint32_t dst = base + rr.s * kStage;
          tma_load_3d(dst, &mapA, kb * BK, row0, ma, bar);                      // A big
          tma_load_4d(dst + kOffBb, &mapB, 0, kb * BK, col0 / 32, mb, bar);     // B big
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------ MMA issuer (leader) ------------------------------
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = tf32_idesc(2 * kRowsCta, kPairN) | (1u << 16);  // B MN-major
      Ring<kStages> pr;
      int lt = 0;
      for (int64_t t = cluster; t < grid.tiles; t += nclusters, ++lt) {
        const int buf = lt & 1;
        mbar_wait(smem_u32(&acc_empty[buf]), (uint32_t)((lt >> 1) & 1) ^ 1u);
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(buf * kPairN);
        for (int kb = 0; kb < nk; ++kb, pr.next()) {
          mbar_wait(smem_u32(&ready[pr.s]), pr.ph);
          tc_fence_after();
          if ((debug & 15) != 2) {
            const uint32_t sb = base + pr.s * kStage;
            const uint64_t dAb = kmaj_sw64(sb), dAs = kmaj_sw64(sb + kOffAs);
            const uint64_t dBb = mnmaj_sw128_32b(sb + kOffBb), dBs = mnmaj_sw128_32b(sb + kOffBs);
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint64_t aadv = (uint64_t)(kk * 32) >> 4;     // 8 TF32 along the 64 B row
              const uint64_t badv = (uint64_t)(kk * 1024) >> 4;   // 8 k rows further
              mma_tf32_pair(acc, dAs + aadv, dBb + badv, idesc, (kb | kk) != 0);
              mma_tf32_pair(acc, dAb + aadv, dBs + badv, idesc, 1);
              mma_tf32_pair(acc, dAb + aadv, dBb + badv, idesc, 1);
            }
          }
          mma_commit_pair(smem_u32(&freed[pr.s]));
        }
        mma_commit_pair(smem_u32(&acc_full[buf]));
      }
    }
    __syncwarp();
  } else if (warp < 2 + kXformWarps) {
    // ------------------------------ transform ------------------------------
    // Thread u = 32 xw + lane owns byte 16u of each operand half: A row u/4 (4 k values),
    // B k-row (u % 128) / 8 of column chunk u / 128 (4 n values). It reads its 16 B of the
    // raw fp32, multiplies by the factor, rounds big to TF32 in place and writes small to
    // the twin plane: contiguous 512 B per warp, the swizzle is irrelevant in place.
    const int xw = warp - 2;
    const int u = xw * 32 + lane;
    const int arow_cta = u >> 2;
    const int bkrow = (u & 127) >> 3;
    const uint32_t ready0 = smem_u32(&ready[0]);
    float* fac = reinterpret_cast<float*>(smem + Y::kFacOff);  // [2][kMaxK]
    Ring<kStages> rr;
    // per-tile factors, fetched one tile ahead: this thread's B row scales for k = u and
    // u + 512 (the tile's table is built from them), its A row's q[row][J]
    float qbn[2], qan[4], gBn = 0.0f;
    // fetch(tile, block): false (nothing read) when block is false and a chained tile's
    // inputs are not complete yet — the look-ahead never waits on a later step
    auto fetch = [&](int64_t tile, bool block) -> bool {
      int64_t b;
      int prow0, pcol0, step;
      decode(tile, b, prow0, pcol0, step);
      const int JB = pcol0 / 256;
      if constexpr (kChain) {
        if (!block && !dep_ready(b, JB, step)) return false;
        dep_wait(b, JB, step);
      }
      const int arow = prow0 + (int)rank * kRowsCta + arow_cta;
      const float* qa = A.q + (kChain ? idx_a(b, step) : b / A.div) * A.sq + (int64_t)arow * nJk;
#pragma unroll
      for (int J = 0; J < 4; ++J) qan[J] = J < nJk ? qa[J] : kNegInf;
      const int64_t ib = kChain ? idx_b(b, step) : b / B.div;
      const float* qb = B.q + ib * B.sq + JB;
#pragma unroll
      for (int h = 0; h < 2; ++h) qbn[h] = u + 512 * h < k ? qb[(int64_t)(u + 512 * h) * nJm] : 0.0f;
      gBn = decode_g(B.G[ib * B.sG + JB]);
      if (clampz) gBn = fmaxf(gBn, 0.0f);  // Eq. 11: b = max(colmax B, 0)
      return true;
    };
    bool fetched = cluster < grid.tiles && fetch(cluster, true);
    int tpar = 0;
    for (int64_t t = cluster; t < grid.tiles; t += nclusters, tpar ^= 1) {
      if (!fetched) fetch(t, true);
      float* ft = fac + tpar * kMaxK;
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (u + 512 * h < k) ft[u + 512 * h] = scale_factor(qbn[h], gBn);
      float qac[4];
#pragma unroll
      for (int J = 0; J < 4; ++J) qac[J] = qan[J];
      float rho = fmaxf(fmaxf(qac[0], qac[1]), fmaxf(qac[2], qac[3]));
      if (clampz) rho = fmaxf(rho, 0.0f);  // Eq. 11: a = max(rowmax A, 0)
      asm volatile("bar.sync 1, %0;" ::"n"(kXformWarps * 32) : "memory");  // table complete
      fetched = t + nclusters < grid.tiles && fetch(t + nclusters, false);
      float fa = 0.0f;
      int curJ = -1;
      for (int kb = 0; kb < nk; ++kb, rr.next()) {
        const int J = (kb * BK) >> 8;
        if (J != curJ) {
          const float qj = J == 0 ? qac[0] : J == 1 ? qac[1] : J == 2 ? qac[2] : qac[3];
          fa = scale_factor(qj, rho);
          curJ = J;
        }
        float fb = ft[kb * BK + bkrow];
        if (debug & 256) fb = 1.0f, fa = 1.0f;  // layout probe: no factors
        mbar_wait(smem_u32(&full[rr.s]), rr.ph);
        const uint32_t sb = base + rr.s * kStage + u * 16;
        const float4 va = ld_shared_v4(sb);
        const float4 vb = ld_shared_v4(sb + kOffBb);
        if (debug & 128) {  // layout probe: all-ones operands
          const uint32_t one = __float_as_uint(1.0f);
          st_shared_v4(sb, one, one, one, one);
          st_shared_v4(sb + kOffAs, 0u, 0u, 0u, 0u);
          st_shared_v4(sb + kOffBb, one, one, one, one);
          st_shared_v4(sb + kOffBs, 0u, 0u, 0u, 0u);
        } else if ((debug & 15) != 1) {
          uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
          split_tf32(va.x * fa, h0, l0);
          split_tf32(va.y * fa, h1, l1);
          split_tf32(va.z * fa, h2, l2);
          split_tf32(va.w * fa, h3, l3);
          st_shared_v4(sb, h0, h1, h2, h3);
          st_shared_v4(sb + kOffAs, l0, l1, l2, l3);
          split_tf32(vb.x * fb, h0, l0);
          split_tf32(vb.y * fb, h1, l1);
          split_tf32(vb.z * fb, h2, l2);
          split_tf32(vb.w * fb, h3, l3);
          st_shared_v4(sb + kOffBb, h0, h1, h2, h3);
          st_shared_v4(sb + kOffBs, l0, l1, l2, l3);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_rank(ready0 + rr.s * 8, 0);
      }
    }
  } else {
    // ------------------------------ epilogue ------------------------------
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t acc_empty0 = smem_u32(&acc_empty[0]);
    constexpr int kOB = Y::kOutBufs > 0 ? Y::kOutBufs : 1;
    const uint32_t obuf = base + kOutOff + (uint32_t)(warp - 2 - kXformWarps) * kOB * kOutStage;
    int lt = 0;
    for (int64_t t = cluster; t < grid.tiles; t += nclusters, ++lt) {
      int64_t b;
      int prow0, pcol0, step;
      decode(t, b, prow0, pcol0, step);
      const int buf = lt & 1;
      const int grow = prow0 + (int)rank * kRowsCta + row;
      const int wrow0 = prow0 + (int)rank * kRowsCta + quad * 32;
      const int JB = pcol0 / 256;
      const int64_t io = idx_o(b, step);
      if constexpr (kChain) dep_wait(b, JB, step);
      // product scales: rowmax q of the left operand's row, G of the right operand's block
      const float* qa = A.q + (kChain ? idx_a(b, step) : b / A.div) * A.sq + (int64_t)grow * nJk;
      float rho = kNegInf;
      for (int J = 0; J < nJk; ++J) rho = fmaxf(rho, qa[J]);
      float gB = decode_g(B.G[(kChain ? idx_b(b, step) : b / B.div) * B.sG + JB]);
      if (clampz) {  // the same clamped scales as the transform (Eq. 11, core.py:252-253)
        rho = fmaxf(rho, 0.0f);
        gB = fmaxf(gB, 0.0f);
      }
      mbar_wait(smem_u32(&acc_full[buf]), (uint32_t)((lt >> 1) & 1));
      tc_fence_after();
      const uint32_t tacc = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * kPairN);
      if constexpr (kOut == kTsOutGoom) {
#pragma unroll 1
        for (int col = 0; col < kPairN; col += 32) {
          uint32_t v[32];
          tmem_ld32(tacc + col, v);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t sbuf = obuf + (uint32_t)(h % kOB) * kOutStage;
            if (lane == 0) tma_store_wait_read<kOB - 1>();
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
              const float2 o0 = tc_out(__uint_as_float(v[16 * h + j]), rho, gB);
              const float2 o1 = tc_out(__uint_as_float(v[16 * h + j + 1]), rho, gB);
              const float2 o2 = tc_out(__uint_as_float(v[16 * h + j + 2]), rho, gB);
              const float2 o3 = tc_out(__uint_as_float(v[16 * h + j + 3]), rho, gB);
              const uint32_t rb = sbuf + (uint32_t)lane * 128;
              st_shared_v4(rb + ((((j >> 1) + 0) ^ (lane & 7)) << 4), __float_as_uint(o0.x),
                           __float_as_uint(o0.y), __float_as_uint(o1.x), __float_as_uint(o1.y));
              st_shared_v4(rb + ((((j >> 1) + 1) ^ (lane & 7)) << 4), __float_as_uint(o2.x),
                           __float_as_uint(o2.y), __float_as_uint(o3.x), __float_as_uint(o3.y));
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) tma_store_3d(&mapOut, sbuf, pcol0 + col + 16 * h, wrow0, (int)b);
          }
        }
      } else {
        // pass 1: max |S| over this row's 256 columns
        float mx = 0.0f;
        bool bad = false;
#pragma unroll 1
        for (int col = 0; col < kPairN; col += 32) {
          uint32_t v[32];
          tmem_ld32(tacc + col, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float a = fabsf(__uint_as_float(v[j]));
            bad |= !(a <= 3.0e38f);  // inf or NaN
            mx = fmaxf(mx, a);
          }
        }
        // exact power-of-two normalisation: mx * 2^-e in [0.5, 1)
        const uint32_t ex = (__float_as_uint(mx) >> 23) & 0xFFu;
        const bool norm = mx > 0.0f && ex >= 2u && ex <= 252u;
        const int e = norm ? (int)ex - 126 : 0;
        const float sc = __uint_as_float((uint32_t)(127 - e) << 23);  // 2^-e
        const float qrow = mx > 0.0f ? __fadd_rn(__fadd_rn(rho, gB), (float)e * kLn2) : kNegInf;
        if constexpr (kOut == kTsOutTs) {
#pragma unroll 1
          for (int col = 0; col < kPairN; col += 32) {
            uint32_t v[32];
            tmem_ld32(tacc + col, v);
            const uint32_t sbuf = obuf + (uint32_t)(((col >> 5) & 1) % kOB) * kOutStage;
            if (lane == 0) tma_store_wait_read<kOB - 1>();
            __syncwarp();
            const uint32_t rb = sbuf + (uint32_t)lane * 128;
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              st_shared_v4(rb + (((j >> 2) ^ (lane & 7)) << 4),
                           __float_as_uint(__uint_as_float(v[j]) * sc),
                           __float_as_uint(__uint_as_float(v[j + 1]) * sc),
                           __float_as_uint(__uint_as_float(v[j + 2]) * sc),
                           __float_as_uint(__uint_as_float(v[j + 3]) * sc));
            fence_async_smem();
            __syncwarp();
            if (lane == 0) tma_store_3d(&mapOut, sbuf, pcol0 + col, wrow0, (int)io);
          }
          T.q[io * T.sq + (int64_t)grow * nJm + JB] = qrow;
          const float gmax = warp_max(qrow);
          if (lane == 0 && gmax != kNegInf)
            atomicMax(&T.G[io * T.sG + JB], float_to_ordered(gmax));
        } else {
          // digest: this row's max log and log Frobenius norm, reduced over the warp's 32 rows
          float ss = 0.0f;
#pragma unroll 1
          for (int col = 0; col < kPairN; col += 32) {
            uint32_t v[32];
            tmem_ld32(tacc + col, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float a = __uint_as_float(v[j]) * sc;
              ss = fmaf(a, a, ss);
            }
          }
          const float lmax = mx > 0.0f ? __fadd_rn(qrow, logf(mx * sc)) : kNegInf;
          const float lfro = mx > 0.0f ? __fadd_rn(qrow, 0.5f * logf(ss)) : kNegInf;
          const float wmax = warp_max(lmax);
          const float top = warp_max(lfro);
          const float w = top == kNegInf ? 0.0f : expf(2.0f * (lfro - top));
          const float sum = warp_sum(w);
          const bool wbad = __any_sync(0xffffffffu, bad || !(rho < INFINITY) || !(gB < INFINITY));
          if (lane == 0)
            parts[(b * (n / 32) + wrow0 / 32) * nJm + JB] =
                make_float4(wmax, top, sum, wbad ? 1.0f : 0.0f);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_rank(acc_empty0 + buf * 8, 0);
      if constexpr (kChain) {  // publish this CTA's part of the output tile (U, q, G) to the next step
        if (lane == 0) {
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        asm volatile("bar.sync 2, %0;" ::"n"(kEpiWarps * 32) : "memory");
        if (warp == 2 + kXformWarps && lane == 0)
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ch.done + b * nJm + JB)
                       : "memory");
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

// GOOM_TS_SCALES=truemax: scale by the operands' true maxima instead of Eq. 11's clamped
// max(rowmax, 0) / max(colmax, 0) (core.py:252-253). Opt-in only: with the clamp a shrinking
// chain underflows to -inf exactly where the reference's float32 run (and this library's
// complex64 kernels) do; without it the engine returns the finite product instead.
int ts_clamp() {
  static int v = [] {
    const char* e = getenv("GOOM_TS_SCALES");
    return (e && std::string(e) == "truemax") ? 0 : 1;
  }();
  return v;
}

int ts_debug() {
  static int v = [] {
    const char* e = getenv("GOOM_TS_DEBUG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// GOOM_TS_PDL=0 launches without programmatic dependent launch (A/B probe)
int ts_pdl() {
  static int v = [] {
    const char* e = getenv("GOOM_TS_PDL");
    return e ? atoi(e) : 1;
  }();
  return v;
}

template <int kOut, int S>
int query_clusters() {
  return [] {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * 74);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Lay<kOut, S>::kSmem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, lmme_ts_kernel<kOut, S, false>, &cfg) != cudaSuccess ||
        n < 1) {
      cudaGetLastError();
      n = num_sms() / 2;
    }
    return n;
  }();
}
template <int kOut, int S>
int max_clusters() {  // per device (abi.cu per_device_value)
  return per_device_value((const void*)lmme_ts_kernel<kOut, S, false>, &query_clusters<kOut, S>);
}

template <int kOut, int S, bool kChain = false>
int launch_cfg(const TsProblem& p, const CUtensorMap& mapA, const CUtensorMap& mapB,
               const CUtensorMap& mapOut, cudaStream_t s) {
  constexpr int kSmem = Lay<kOut, S>::kSmem;
  GOOM_TRY(smem_attr((const void*)lmme_ts_kernel<kOut, S, kChain>, kSmem,
                     "lmme_ts smem attribute"));
  PairGrid pg;
  pg.nct = p.m / kPairN;
  pg.nrt = p.n / 256;
  pg.tiles = p.batch * pg.nct * pg.nrt;
  ChainArgs ch{p.chain_done, p.chain_s, pg.tiles};
  if (p.chain_s) pg.tiles *= p.chain_s - 1;  // every step of the block chains, step-major
  const int64_t mc = max_clusters<kOut, S>();
  const int64_t clusters = pg.tiles < mc ? pg.tiles : mc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * clusters));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  const int pdl = ts_pdl();
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  cudaLaunchKernelEx(&cfg, lmme_ts_kernel<kOut, S, kChain>, mapA, mapB, mapOut, p.A, p.B, p.T,
                     p.parts, pg,
                     p.n, p.k, p.m, ts_debug(), ch, ts_clamp(), pdl);
  GOOM_CHECK_LAUNCH("lmme_ts_kernel");
  return GOOM_OK;
}

// ring depths (raw, plane): GOOM_TS_STAGES=<index> picks a probe configuration
int stage_cfg() {
  static int v = [] {
    const char* e = getenv("GOOM_TS_STAGES");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <int kOut>
int launch(const TsProblem& p, const CUtensorMap& mapA, const CUtensorMap& mapB,
           const CUtensorMap& mapOut, cudaStream_t s) {
  if constexpr (kOut == kTsOutDigest) {
    if (stage_cfg() == 1) return launch_cfg<kOut, 5>(p, mapA, mapB, mapOut, s);
    return launch_cfg<kOut, 6>(p, mapA, mapB, mapOut, s);
  } else {
    if constexpr (kOut == kTsOutTs)
      if (p.chain_s) return launch_cfg<kOut, 5, true>(p, mapA, mapB, mapOut, s);
    if (stage_cfg() == 1) return launch_cfg<kOut, 4>(p, mapA, mapB, mapOut, s);
    if (stage_cfg() == 2) return launch_cfg<kOut, 6>(p, mapA, mapB, mapOut, s);
    return launch_cfg<kOut, 5>(p, mapA, mapB, mapOut, s);
  }
}

inline int64_t mats(int64_t stride, int64_t div, int64_t batch) {
  return stride == 0 ? 1 : (batch - 1) / div + 1;
}

}  // namespace

bool lmme_ts_eligible(int n, int k, int m) {
  // k <= 1024: the transform keeps a tile's per-K-block factors in two registers per lane
  return n > 0 && k > 0 && m > 0 && n % 256 == 0 && k % 256 == 0 && m % 256 == 0 && k <= 1024;
}

int lmme_ts(const TsProblem& p, cudaStream_t s) {
  if (!lmme_ts_eligible(p.n, p.k, p.m)) return fail(GOOM_EUNSUPPORTED, "lmme_ts: n, k, m % 256");
  if (p.batch == 0) return GOOM_OK;
  if (p.chain_s && (p.kind != kTsOutTs || p.n != p.k || !p.chain_done || p.chain_s < 2 ||
                    p.chain_T < p.batch * p.chain_s))
    return fail(GOOM_EINVAL, "lmme_ts: chained phase 1 needs a square tile-scaled output");
  // matrices each map spans: a chained launch addresses every matrix of its buffers
  const int64_t nA = p.chain_s ? p.chain_T : mats(p.A.sU, p.A.div, p.batch);
  const int64_t nB = p.chain_s ? p.chain_T : mats(p.B.sU, p.B.div, p.batch);
  const uintptr_t al = reinterpret_cast<uintptr_t>(p.A.U) | reinterpret_cast<uintptr_t>(p.B.U);
  if ((al & 15) || ((p.A.sU | p.B.sU) & 3)) return fail(GOOM_EINVAL, "lmme_ts: operand alignment");
  alignas(64) CUtensorMap mapA, mapB, mapOut;
  {  // A fp32 (k, n, matrix), box 16 k x 128 rows, 64B swizzle: the UMMA K-major SW64 layout
    cuuint64_t dims[3] = {(cuuint64_t)p.k, (cuuint64_t)p.n, (cuuint64_t)nA};
    cuuint64_t strides[2] = {(cuuint64_t)p.k * 4,
                             (cuuint64_t)(p.A.sU ? p.A.sU : (int64_t)p.n * p.k) * 4};
    cuuint32_t box[3] = {BK, kRowsCta, 1};
    GOOM_TRY(encode_raw(&mapA, p.A.U, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dims, strides, box,
                        CU_TENSOR_MAP_SWIZZLE_64B));
  }
  {  // B fp32 (32 cols, k, m/32 chunks, matrix), box 32 x 16 k x 4 x 1, 128B/32B-atom
     // swizzle: [chunk][k][32 cols] = the UMMA MN-major 128B_BASE32B layout (chunks 2 KB apart)
    cuuint64_t dims[4] = {32, (cuuint64_t)p.k, (cuuint64_t)(p.m / 32), (cuuint64_t)nB};
    cuuint64_t strides[3] = {(cuuint64_t)p.m * 4, 128,
                             (cuuint64_t)(p.B.sU ? p.B.sU : (int64_t)p.k * p.m) * 4};
    cuuint32_t box[4] = {32, BK, kPairN / 2 / 32, 1};
    GOOM_TRY(encode_raw(&mapB, p.B.U, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dims, strides, box,
                        CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B));
  }
  if (p.kind == kTsOutGoom) {
    if ((reinterpret_cast<uintptr_t>(p.C) & 15) || (p.strideC & 1))
      return fail(GOOM_EINVAL, "lmme_ts: output alignment");
    const int64_t cb = p.strideC == 0 ? 1 : p.batch;
    const int64_t cs = p.strideC == 0 ? (int64_t)p.n * p.m : p.strideC;
    cuuint64_t dims[3] = {(cuuint64_t)p.m, (cuuint64_t)p.n, (cuuint64_t)cb};
    cuuint64_t strides[2] = {(cuuint64_t)p.m * 8, (cuuint64_t)cs * 8};
    cuuint32_t box[3] = {16, 32, 1};
    GOOM_TRY(encode_raw(&mapOut, p.C, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, dims, strides, box,
                        CU_TENSOR_MAP_SWIZZLE_128B));
    return launch<kTsOutGoom>(p, mapA, mapB, mapOut, s);
  }
  if (p.kind == kTsOutTs) {
    if ((reinterpret_cast<uintptr_t>(p.T.U) & 15) || (p.T.sU & 3))
      return fail(GOOM_EINVAL, "lmme_ts: output alignment");
    const int64_t cb = p.chain_s ? p.chain_T : (p.T.sU == 0 ? 1 : p.batch);
    const int64_t cs = p.T.sU == 0 ? (int64_t)p.n * p.m : p.T.sU;
    cuuint64_t dims[3] = {(cuuint64_t)p.m, (cuuint64_t)p.n, (cuuint64_t)cb};
    cuuint64_t strides[2] = {(cuuint64_t)p.m * 4, (cuuint64_t)cs * 4};
    cuuint32_t box[3] = {32, 32, 1};
    GOOM_TRY(encode_raw(&mapOut, p.T.U, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dims, strides, box,
                        CU_TENSOR_MAP_SWIZZLE_128B));
    return launch<kTsOutTs>(p, mapA, mapB, mapOut, s);
  }
  mapOut = mapA;  // unused by the digest epilogue
  return launch<kTsOutDigest>(p, mapA, mapB, mapOut, s);
}

// ---- conversions ------------------------------------------------------------------

namespace {

// one warp per (matrix, row, 256-column block): q = max log (clamped below by nothing: the
// block's own maximum), U = sign * exp(log - q); G via ordered atomicMax
__global__ void goom_to_ts_kernel(const float2* __restrict__ X, int64_t sX, TsOut out,
                                  int64_t batch, int rows, int cols) {
  const int nJ = cols / 256;
  const int64_t units = batch * rows * nJ;
  const int lane = threadIdx.x & 31;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < units;
       u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int J = (int)(u % nJ);
    const int64_t r = (u / nJ) % rows;
    const int64_t b = u / ((int64_t)nJ * rows);
    const float2* x = X + b * sX + r * cols + J * 256;
    float2 v[8];
    float mx = kNegInf;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i] = x[i * 32 + lane];
      mx = fmaxf(mx, v[i].x);
    }
    mx = warp_max(mx);
    float* U = out.U + b * out.sU + r * cols + J * 256;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float e = mx == kNegInf ? 0.0f : expf(v[i].x - mx);
      U[i * 32 + lane] = phase_negative(v[i].y) ? -e : e;
    }
    if (lane == 0) {
      out.q[b * out.sq + r * nJ + J] = mx;
      if (mx != kNegInf) atomicMax(&out.G[b * out.sG + J], float_to_ordered(mx));
    }
  }
}

__global__ void ts_to_goom_kernel(TsIn in, float2* __restrict__ X, int64_t sX, int64_t batch,
                                  int rows, int cols) {
  const int nJ = cols / 256;
  const int64_t n = batch * rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % cols);
    const int64_t r = (i / cols) % rows;
    const int64_t b = i / ((int64_t)cols * rows);
    const int64_t mb = b / in.div;
    const float u = in.U[mb * in.sU + r * cols + c];
    const float q = in.q[mb * in.sq + r * nJ + c / 256];
    X[b * sX + r * cols + c] = make_float2(u == 0.0f ? kNegInf : __fadd_rn(logf(fabsf(u)), q),
                                           u < 0.0f ? kPi : 0.0f);
  }
}

// per matrix: combine (max log, lfro top, sum e^{2(lfro - top)}, bad) partials
__global__ void digest_reduce_kernel(const float4* __restrict__ parts, int per,
                                     float4* __restrict__ out, int64_t batch) {
  const int64_t b = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= batch) return;
  const float4* p = parts + b * per;
  float mx = kNegInf, top = kNegInf;
  bool bad = false;
  for (int i = lane; i < per; i += 32) {
    mx = fmaxf(mx, p[i].x);
    top = fmaxf(top, p[i].y);
    bad |= p[i].w != 0.0f;
  }
  mx = warp_max(mx);
  top = warp_max(top);
  float s = 0.0f;
  if (top != kNegInf)
    for (int i = lane; i < per; i += 32)
      if (p[i].y != kNegInf) s += p[i].z * expf(2.0f * (p[i].y - top));
  s = warp_sum(s);
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0)
    out[b] = make_float4(mx, top == kNegInf ? kNegInf : top + 0.5f * logf(s),
                         bad || !(mx < INFINITY) ? 0.0f : 1.0f, 0.0f);
}

int grid_for(int64_t threads) {
  int64_t b = (threads + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

int launch_goom_to_ts(const float2* X, int64_t strideX, TsOut out, int64_t batch, int rows,
                      int cols, cudaStream_t s) {
  if (cols % 256) return fail(GOOM_EUNSUPPORTED, "tile-scaled format needs cols % 256 == 0");
  goom_to_ts_kernel<<<grid_for(batch * rows * (cols / 256) * 32), 256, 0, s>>>(X, strideX, out,
                                                                                batch, rows, cols);
  GOOM_CHECK_LAUNCH("goom_to_ts_kernel");
  return GOOM_OK;
}

int launch_ts_to_goom(TsIn in, float2* X, int64_t strideX, int64_t batch, int rows, int cols,
                      cudaStream_t s) {
  ts_to_goom_kernel<<<grid_for(batch * rows * cols), 256, 0, s>>>(in, X, strideX, batch, rows,
                                                                   cols);
  GOOM_CHECK_LAUNCH("ts_to_goom_kernel");
  return GOOM_OK;
}

int launch_digest_reduce(const float4* parts, int parts_per, float4* out, int64_t batch,
                         cudaStream_t s) {
  const int blocks = (int)((batch + 7) / 8);
  digest_reduce_kernel<<<blocks, 256, 0, s>>>(parts, parts_per, out, batch);
  GOOM_CHECK_LAUNCH("digest_reduce_kernel");
  return GOOM_OK;
}

}  // namespace goom
