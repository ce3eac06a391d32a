// Long-chain fold for d = 64 complex64 on tcgen05: the R- and S-passes of the reduce-then-
// scan in scan_long.cu (same tree, same carry contract) with every combine P <- A_t (x) P on
// the tensor cores instead of a lane group's FP32 FMAs.
//
// Two chains share one CTA and one MMA: A = [leaf of chain 0 ; leaf of chain 1] (128 x 64),
// B = [state of chain 0 | state of chain 1] (64 x 128), D = A B (128 x 128 FP32 in TMEM, 3xTF32
// like lmme_tc.cu); the two diagonal 64 x 64 blocks are the new states, the two cross blocks
// are dropped (free: the step is latency-bound, not tensor-bound). Per step:
//   warp 0      TMA: the next leaf pair (raw complex64, 4 K-blocks x 2 chains of [64 x 16])
//               into the other A buffer (double-buffered, 64 KB each);
//   warps 2-9   leaf transform in place: clamped row scale a_i = max(rowmax, 0) (Eq. 11,
//               core.py:252-253), sign * exp(x - a_i) -> (big, small) TF32 planes in the
//               64B-swizzled K-major layout (the same as lmme_tc.cu's A operand);
//   warp 1      24 MMAs (4 K-blocks x 2 x small*big + big*small + big*big), commit;
//   warps 10-13 epilogue, thread = state row i of chain h = i / 64: the accumulator row's
//               64 diagonal columns; output log = (log|acc| + a_i) + Q_h (the LMME epilogue
//               order, core.py:259) and sign; next right operand B_kj = U_j g_i with
//               U = acc 2^-e_i (exact; e_i the row maximum's binary exponent) and
//               g_i = exp((Q_h - Q'_h) + a_i + e_i ln2) <= 2 (the difference of the two state
//               scales first: no rounding at the magnitude of the chain's logs), Q'_h = max(max_i log max_j
//               |x_ij|, 0) is the clamped maximum over the whole new state: the right
//               operand's scale is one value per state (the tile-scaled engine's per-block
//               scale, lmme_ts.cu), not per column — a state column more than ~e^87 below the
//               state's largest entry flushes, as there. The B planes are written K-major
//               (one 4-byte word per (k, n); lanes 16-31 one column ahead: conflict-free).
// Prefixes (S-pass) or chain totals (R-pass) leave through a 128B-swizzled staging buffer per
// epilogue warp and TMA stores. A chain without a carry starts from its first leaf (raw,
// canonical signs), exactly as scan_long.cu.
#include "tc_ptx.cuh"

namespace goom {

namespace {
using namespace tc;

constexpr int kD = 64;
constexpr int kXW = 8;                               // leaf-transform warps
constexpr int kEW = 4;                               // epilogue warps (one per TMEM quadrant)
constexpr int kThreads = 64 + (kXW + kEW) * 32;      // 448
constexpr int kKB = 16384;                           // one K-block of A or B: 16 groups x 1 KB
constexpr int kAbuf = 4 * kKB;                       // a leaf pair: 64 KB
constexpr int kBoff = 2 * kAbuf;                     // B planes (64 KB)
constexpr int kOutOff = kBoff + 4 * kKB;             // staging: 4 warps x [32 rows][32 cols]
constexpr int kWarpOut = 8192;                       //   two 128B-swizzled boxes of 16 columns
constexpr int kRsOff = kOutOff + kEW * kWarpOut;     // leaf row scales [2][128]
constexpr int kQxOff = kRsOff + 2 * 128 * 4;         // per-warp maxima [2 parities][4 warps]
constexpr int kBarOff = kQxOff + 64;
constexpr int kSmem = kBarOff + 128 + 1024;          // + barriers, + 1 KB alignment slack
static_assert(kSmem <= 232448, "shared memory budget");

#ifdef GOOM_L64_TRACE
// profiling build only (tools/tc_trace.sh): clock64 stamps of CTA 0's first 256 steps
__device__ long long g_l64_trace[8][256];
#define L64_TRACE(row, i, v) \
  do {                       \
    if (blockIdx.x == 0 && (i) < 256) g_l64_trace[row][i] = (v); \
  } while (0)
#else
#define L64_TRACE(row, i, v) \
  do {                       \
  } while (0)
#endif

__device__ __forceinline__ float2 canon(float2 z) {
  z.y = phase_negative(z.y) ? kPi : 0.0f;
  return z;
}

// byte offset of TF32 (k, n) in a K-major 64B-swizzled operand of N = 128 (lmme_tc.cu's B
// layout: per K-block 16 groups of 8 n-rows x 16 k, big plane at +0, small at +512)
__device__ __forceinline__ uint32_t kmaj_off(int k, int n) {
  const int r = n & 7, c = (k & 15) >> 2;
  return (uint32_t)((k >> 4) * kKB + (n >> 3) * kGroupBytes + sw64_off(r, c) + (k & 3) * 4);
}

struct FoldArgs {
  const float2* A;        // leaves (T, 64, 64)
  int64_t T, s;           // chain k: leaves [k s, min(k s + s, T))
  const float2* carry0;   // chain 0's right carry (null: start from its first leaf)
  const float2* carries;  // chain k >= 1: carries[k - 1] (null: first leaf)
  float2* out;            // every prefix (S-pass) or null
  float2* tot;            // every chain's last state (R-pass) or null
  int64_t nchains;
};

// per chain of a pair: where it starts and how many combines it runs
struct ChainAt {
  int64_t t0, t1;   // leaves [t0, t1)
  const float2* cin;
  bool live;        // the chain exists
  __device__ __forceinline__ int64_t first() const { return cin ? t0 : t0 + 1; }
  __device__ __forceinline__ int64_t steps() const { return live ? t1 - first() : 0; }
};
__device__ __forceinline__ ChainAt chain_at(const FoldArgs& a, int64_t c) {
  ChainAt r;
  r.live = c < a.nchains;
  r.t0 = c * a.s;
  r.t1 = r.t0 + a.s < a.T ? r.t0 + a.s : a.T;
  r.cin = !r.live ? nullptr : (c == 0 ? a.carry0 : (a.carries ? a.carries + (c - 1) * kD * kD : nullptr));
  return r;
}

__global__ void __launch_bounds__(kThreads, 1)
    long_fold64_kernel(const __grid_constant__ CUtensorMap mapA,
                       const __grid_constant__ CUtensorMap mapO, FoldArgs fa, int64_t npairs) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t base = smem_u32(smem);
  float* rS = reinterpret_cast<float*>(smem + kRsOff);    // [buf][128]
  float* Qx = reinterpret_cast<float*>(smem + kQxOff);    // [parity][4 warps]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
  uint64_t* a_full = bars;        // [2] leaf pair landed (tx bytes)
  uint64_t* a_ready = bars + 2;   // [2] leaf pair transformed (8 warps)
  uint64_t* a_free = bars + 4;    // [2] the MMAs reading the buffer retired (commit)
  uint64_t* rs_free = bars + 6;   // [2] the epilogue read the buffer's row scales (4 warps)
  uint64_t* b_ready = bars + 8;   // B planes of the next step written (4 warps)
  uint64_t* acc_full = bars + 9;  // accumulator complete (commit)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&a_full[i]), 1);
      mbar_init(smem_u32(&a_ready[i]), kXW);
      mbar_init(smem_u32(&a_free[i]), 1);
      mbar_init(smem_u32(&rs_free[i]), kEW);
    }
    mbar_init(smem_u32(b_ready), kEW);
    mbar_init(smem_u32(acc_full), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------ loader ------------------------------
    if (lane == 0) {
      int64_t g = 0;  // global step (A buffer g & 1)
      for (int64_t p = blockIdx.x; p < npairs; p += gridDim.x) {
        const ChainAt c0 = chain_at(fa, 2 * p), c1 = chain_at(fa, 2 * p + 1);
        const int64_t n = max(c0.steps(), c1.steps());
        for (int64_t j = 0; j < n; ++j, ++g) {
          const int buf = (int)(g & 1);
          if (g >= 2) mbar_wait(smem_u32(&a_free[buf]), (uint32_t)(((g >> 1) - 1) & 1));
          const int64_t l0 = c0.first() + j, l1 = c1.first() + j;
          const bool v0 = j < c0.steps(), v1 = j < c1.steps();
          const uint32_t bar = smem_u32(&a_full[buf]);
          mbar_expect_tx(bar, (uint32_t)((v0 ? 1 : 0) + (v1 ? 1 : 0)) * (kAbuf / 2));
          const uint32_t dst = base + (uint32_t)buf * kAbuf;
#pragma unroll
          for (int kb = 0; kb < 4; ++kb) {  // [64 rows][16 k] boxes: groups 0-7 | 8-15
            if (v0) tma_load_3d(dst + kb * kKB, &mapA, kb * 16, 0, (int)l0, bar);
            if (v1) tma_load_3d(dst + kb * kKB + kKB / 2, &mapA, kb * 16, 0, (int)l1, bar);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ------------------------------
    if (lane == 0) {
      constexpr uint32_t idesc = tf32_idesc(128, 128);
      int64_t g = 0, bw = 0;
      for (int64_t p = blockIdx.x; p < npairs; p += gridDim.x) {
        const ChainAt c0 = chain_at(fa, 2 * p), c1 = chain_at(fa, 2 * p + 1);
        const int64_t n = max(c0.steps(), c1.steps());
        for (int64_t j = 0; j < n; ++j, ++g, ++bw) {
          const int buf = (int)(g & 1);
          mbar_wait(smem_u32(&a_ready[buf]), (uint32_t)((g >> 1) & 1));
          L64_TRACE(0, g, clock64());
          mbar_wait(smem_u32(b_ready), (uint32_t)(bw & 1));
          tc_fence_after();
          L64_TRACE(1, g, clock64());
#pragma unroll
          for (int kb = 0; kb < 4; ++kb) {
            const uint32_t sa = base + (uint32_t)buf * kAbuf + kb * kKB, sb = base + kBoff + kb * kKB;
            const uint64_t dAb = sw64_desc(sa), dAs = sw64_desc(sa + 512);
            const uint64_t dBb = sw64_desc(sb), dBs = sw64_desc(sb + 512);
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              const uint64_t adv = (uint64_t)(kk * 32) >> 4;
              mma_tf32(tmem, dAs + adv, dBb + adv, idesc, (kb | kk) != 0);
              mma_tf32(tmem, dAb + adv, dBs + adv, idesc, 1);
              mma_tf32(tmem, dAb + adv, dBb + adv, idesc, 1);
            }
          }
          mma_commit(smem_u32(&a_free[buf]));
          mma_commit(smem_u32(acc_full));
        }
      }
    }
    __syncwarp();
  } else if (warp < 2 + kXW) {
    // ------------------------------ leaf transform ------------------------------
    // warp w: rows 16 w .. 16 w + 15 = groups 2w, 2w + 1 of every K-block; lane: rows
    // (lane >> 3) and 4 + (lane >> 3) of each group, k-pair lane & 7 (lmme_tc.cu's A side)
    const int w = warp - 2, r = lane >> 3, kp = lane & 7;
    const int h = w >> 2;  // chain of these rows
    int64_t g = 0;
    for (int64_t p = blockIdx.x; p < npairs; p += gridDim.x) {
      const ChainAt c0 = chain_at(fa, 2 * p), c1 = chain_at(fa, 2 * p + 1);
      const int64_t n = max(c0.steps(), c1.steps());
      const int64_t mysteps = h ? c1.steps() : c0.steps();
      for (int64_t j = 0; j < n; ++j, ++g) {
        const int buf = (int)(g & 1);
        const uint32_t ab = base + (uint32_t)buf * kAbuf;
        mbar_wait(smem_u32(&a_full[buf]), (uint32_t)((g >> 1) & 1));
        if (w == 0 && lane == 0) L64_TRACE(6, g, clock64());
        const bool valid = j < mysteps;
        float sc[4] = {0.f, 0.f, 0.f, 0.f};  // rows (group 2w: r, r+4), (group 2w+1: r, r+4)
        if (valid) {
#pragma unroll
          for (int q = 0; q < 4; ++q) sc[q] = kNegInf;
#pragma unroll
          for (int kb = 0; kb < 4; ++kb)
#pragma unroll
            for (int gg = 0; gg < 2; ++gg) {
              const uint32_t ga = ab + kb * kKB + (2 * w + gg) * kGroupBytes;
              const float4 a0 = ld_shared_v4(ga + lane * 16), a1 = ld_shared_v4(ga + 512 + lane * 16);
              sc[2 * gg] = fmaxf(sc[2 * gg], fmaxf(a0.x, a0.z));
              sc[2 * gg + 1] = fmaxf(sc[2 * gg + 1], fmaxf(a1.x, a1.z));
            }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) sc[q] = fmaxf(sc[q], __shfl_xor_sync(0xffffffffu, sc[q], o));
            sc[q] = fmaxf(sc[q], 0.0f);  // Eq. 11 clamp
          }
        }
        // the epilogue of step g - 2 has read this buffer's row scales
        if (g >= 2) mbar_wait(smem_u32(&rs_free[buf]), (uint32_t)(((g >> 1) - 1) & 1));
        if (kp == 0) {
          float* rs = rS + buf * 128 + 16 * w;
          rs[r] = sc[0];
          rs[r + 4] = sc[1];
          rs[8 + r] = sc[2];
          rs[8 + r + 4] = sc[3];
        }
#pragma unroll
        for (int kb = 0; kb < 4; ++kb)
#pragma unroll
          for (int gg = 0; gg < 2; ++gg) {
            const uint32_t ga = ab + kb * kKB + (2 * w + gg) * kGroupBytes;
            uint32_t hb[4], lb[4];
            if (valid) {
              const float4 a0 = ld_shared_v4(ga + lane * 16), a1 = ld_shared_v4(ga + 512 + lane * 16);
              goom_split<false>(make_float2(a0.x, a0.y), sc[2 * gg], hb[0], lb[0]);
              goom_split<false>(make_float2(a0.z, a0.w), sc[2 * gg], hb[1], lb[1]);
              goom_split<false>(make_float2(a1.x, a1.y), sc[2 * gg + 1], hb[2], lb[2]);
              goom_split<false>(make_float2(a1.z, a1.w), sc[2 * gg + 1], hb[3], lb[3]);
            } else {  // a finished chain multiplies by the identity (its output is dropped)
              const int row = (16 * w + 8 * gg + r) & 63, k0 = kb * 16 + 2 * kp;
              hb[0] = row == k0 ? 0x3f800000u : 0u;
              hb[1] = row == k0 + 1 ? 0x3f800000u : 0u;
              hb[2] = row + 4 == k0 ? 0x3f800000u : 0u;
              hb[3] = row + 4 == k0 + 1 ? 0x3f800000u : 0u;
              lb[0] = lb[1] = lb[2] = lb[3] = 0u;
            }
            __syncwarp();  // the group is in registers before it is overwritten
            const uint32_t o0 = sw64_off(r, kp >> 1) + (kp & 1) * 8;
            const uint32_t o1 = sw64_off(r + 4, kp >> 1) + (kp & 1) * 8;
            st_shared_v2(ga + o0, hb[0], hb[1]);
            st_shared_v2(ga + 512 + o0, lb[0], lb[1]);
            st_shared_v2(ga + o1, hb[2], hb[3]);
            st_shared_v2(ga + 512 + o1, lb[2], lb[3]);
          }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&a_ready[buf]));
        if (w == 0 && lane == 0) L64_TRACE(7, g, clock64());
      }
    }
  } else {
    // ------------------------------ epilogue / state ------------------------------
    const int e = warp - 2 - kXW;
    const int quad = warp & 3, i = quad * 32 + lane;  // tile row (TMEM lane)
    const int h = quad >> 1, k = i & 63;               // chain, state row
    const int hw = quad & 1;                            // this warp's half of the chain
    const uint32_t stage = base + kOutOff + (uint32_t)e * kWarpOut;
    const uint32_t bplane = base + kBoff;
    int64_t g = 0, par = 0;  // global step; reduction parity
    // chain max of v over its 64 rows (two warps), clamped at 0
    auto chain_max = [&](float v) {
      v = warp_max(v);
      if (lane == 0) Qx[(par & 1) * 4 + quad] = v;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + h) : "memory");
      const float q = fmaxf(fmaxf(Qx[(par & 1) * 4 + 2 * h], Qx[(par & 1) * 4 + 2 * h + 1]), 0.0f);
      ++par;
      return q;
    };
    // this thread's state row as the next right operand: B[k][64 h + n] = f(n) (lanes 16-31
    // take the columns in pair-swapped order: k and k + 16 share banks, n and n ^ 1 do not)
    auto write_b = [&](auto f) {
#pragma unroll
      for (int jj = 0; jj < 64; ++jj) {
        const bool sw = lane >= 16;
        const float x = sw ? f(jj ^ 1) : f(jj);
        const uint32_t big = tf32_round(x), small = __float_as_uint(x - __uint_as_float(big));
        const uint32_t off = kmaj_off(k, 64 * h + (jj ^ (sw ? 1 : 0)));
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(bplane + off), "r"(big) : "memory");
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(bplane + off + 512), "r"(small) : "memory");
      }
    };
    // stage this warp's 32 rows x 64 columns (o(n): complex64 of column n) of matrix `mat`
    // and TMA-store them: two rounds of two 128B-swizzled [32 rows][16 cols] boxes
    auto store_rows = [&](auto o, int64_t mat) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        if (lane == 0) tma_store_wait_read<0>();
        __syncwarp();
#pragma unroll
        for (int bx = 0; bx < 2; ++bx)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float2 p0 = o(32 * half + 16 * bx + 2 * c), p1 = o(32 * half + 16 * bx + 2 * c + 1);
            st_shared_v4(stage + bx * 4096 + lane * 128 + ((c ^ (lane & 7)) << 4),
                         __float_as_uint(p0.x), __float_as_uint(p0.y), __float_as_uint(p1.x),
                         __float_as_uint(p1.y));
          }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&mapO, stage, 32 * half, 32 * hw, (int)mat);
          tma_store_3d(&mapO, stage + 4096, 32 * half + 16, 32 * hw, (int)mat);
        }
        __syncwarp();
      }
    };
    // a row of 64 complex64 straight to global (once per chain: raw first leaves, totals)
    auto put_row = [&](float2* dst, auto o) {
      float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const float2 a0 = o(2 * q), a1 = o(2 * q + 1);
        d4[q] = make_float4(a0.x, a0.y, a1.x, a1.y);
      }
    };
    for (int64_t p = blockIdx.x; p < npairs; p += gridDim.x) {
      const ChainAt c0 = chain_at(fa, 2 * p), c1 = chain_at(fa, 2 * p + 1);
      const ChainAt& cm = h ? c1 : c0;
      const int64_t n = max(c0.steps(), c1.steps());
      const int64_t mysteps = cm.steps();
      // initial state: the carry, or the chain's first leaf (raw), or the identity for a
      // chain that does not exist; Q = its clamped maximum log
      float Q;
      {
        const float2* src = cm.live ? (cm.cin ? cm.cin : fa.A + cm.t0 * kD * kD) : nullptr;
        const float2* srow = src ? src + k * kD : nullptr;
        float m = kNegInf;
        if (srow) {
#pragma unroll 8
          for (int q = 0; q < 64; ++q) m = fmaxf(m, __ldg(&srow[q].x));
        }
        Q = chain_max(srow ? m : 0.0f);
        if (srow) {
          const float Qi = Q;
          write_b([&](int q) {
            const float2 z = __ldg(&srow[q]);
            const float ex = ex2_approx(__fsub_rn(z.x, Qi) * kLog2e);
            return phase_negative(z.y) ? -ex : ex;
          });
        } else {
          write_b([&](int q) { return q == k ? 1.0f : 0.0f; });
        }
        if (cm.live && !cm.cin) {  // the first leaf is the chain's first prefix (raw)
          auto rawc = [&](int q) { return canon(__ldg(&srow[q])); };
          if (fa.out) put_row(fa.out + cm.t0 * kD * kD + k * kD, rawc);
          if (fa.tot && cm.t1 - cm.t0 == 1) put_row(fa.tot + (2 * p + h) * kD * kD + k * kD, rawc);
        }
        fence_async_smem();
        __syncwarp();
        if (n > 0 && lane == 0) mbar_arrive(smem_u32(b_ready));
      }
      for (int64_t j = 0; j < n; ++j, ++g) {
        const int buf = (int)(g & 1);
        mbar_wait(smem_u32(acc_full), (uint32_t)(g & 1));
        tc_fence_after();
        if (e == 0 && lane == 0) L64_TRACE(2, g, clock64());
        const float a = rS[buf * 128 + i];
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&rs_free[buf]));
        uint32_t acc[64];
        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(64 * h),
                  *reinterpret_cast<uint32_t(*)[32]>(&acc[0]));
        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(64 * h + 32),
                  *reinterpret_cast<uint32_t(*)[32]>(&acc[32]));
        const bool valid = j < mysteps;
        const bool more = j + 1 < n;
        // new state: row maximum, its binary exponent, the clamped chain maximum log
        float m = 0.0f;
#pragma unroll
        for (int q = 0; q < 64; ++q) m = fmaxf(m, fabsf(__uint_as_float(acc[q])));
        if (!(m >= 1.17549435e-38f)) m = 0.0f;  // subnormal rows (and NaN) leave the state
        const float lmax = m > 0.0f ? __fadd_rn(__fadd_rn(fast_log_abs(m), a), Q) : kNegInf;
        if (e == 0 && lane == 0) L64_TRACE(3, g, clock64());
        const float Qn = chain_max(valid ? lmax : kNegInf);
        if (e == 0 && lane == 0) L64_TRACE(4, g, clock64());
        if (more) {
          if (valid && m > 0.0f) {
            const int ex = ((__float_as_int(m) >> 23) & 0xff) - 126;  // m = f 2^ex, f in [0.5, 1)
            const float scale = __int_as_float((127 - ex) << 23);    // 2^-ex, exact
            // exponent of the factor at small magnitude: Q - Qn first (both ~ the state's log
            // scale, exact by Sterbenz), then a and ex ln2 — (a + Q) - Qn would round at |Q|
            const float gfac = ex2_approx(
                __fadd_rn(__fadd_rn(__fsub_rn(Q, Qn), a), (float)ex * kLn2) * kLog2e);
            write_b([&](int q) { return (__uint_as_float(acc[q]) * scale) * gfac; });
          } else if (valid) {
            write_b([&](int q) { return 0.0f; });
          } else {  // a finished chain keeps the identity (its products are dropped)
            write_b([&](int q) { return q == k ? 1.0f : 0.0f; });
          }
          fence_async_smem();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(b_ready));
          if (e == 0 && lane == 0) L64_TRACE(5, g, clock64());
        }
        // outputs: every prefix (S-pass), the chain's last state (R-pass)
        auto outc = [&](int q) { return tc_out(__uint_as_float(acc[q]), a, Q); };
        if (valid && fa.out) store_rows(outc, cm.first() + j);
        if (valid && fa.tot && j + 1 == mysteps) put_row(fa.tot + (2 * p + h) * kD * kD + k * kD, outc);
        Q = Qn;
        tc_fence_before();
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
  }
}

}  // namespace

int launch_fold64(const float2* A, int64_t T, int64_t s, const float2* carry0,
                  const float2* carries, float2* out, float2* tot, cudaStream_t st) {
  GOOM_TRY(smem_attr((const void*)long_fold64_kernel, kSmem, "long_fold64 smem"));
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (out && (reinterpret_cast<uintptr_t>(out) & 15)) ||
      (tot && (reinterpret_cast<uintptr_t>(tot) & 15)))
    return fail(GOOM_EUNSUPPORTED, "long_fold64: 16-byte aligned tensors");
  alignas(64) CUtensorMap mapA, mapO;
  {  // leaves (k, row, matrix) complex64 as int64, box 16 k x 64 rows
    cuuint64_t dims[3] = {64, 64, (cuuint64_t)T};
    cuuint64_t strides[2] = {64 * 8, 64 * 64 * 8};
    cuuint32_t box[3] = {16, 64, 1};
    GOOM_TRY(encode(&mapA, Operand{A, 0, 1}, 3, dims, strides, box));
  }
  if (out) {  // prefixes (col, row, matrix), box 16 cols x 32 rows, 128B swizzle
    cuuint64_t dims[3] = {64, 64, (cuuint64_t)T};
    cuuint64_t strides[2] = {64 * 8, 64 * 64 * 8};
    cuuint32_t box[3] = {16, 32, 1};
    GOOM_TRY(encode(&mapO, Operand{out, 0, 1}, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B));
  } else {
    mapO = mapA;  // unused
  }
  FoldArgs fa{A, T, s, carry0, carries, out, tot, (T + s - 1) / s};
  const int64_t npairs = (fa.nchains + 1) / 2;
  const int64_t sms = num_sms();
  const unsigned grid = (unsigned)(npairs < sms ? npairs : sms);
  long_fold64_kernel<<<grid, kThreads, kSmem, st>>>(mapA, mapO, fa, npairs);
  GOOM_CHECK_LAUNCH("long_fold64_kernel");
  return GOOM_OK;
}

}  // namespace goom

#ifdef GOOM_L64_TRACE
extern "C" int goom_l64_trace_read(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, goom::g_l64_trace, sizeof(goom::g_l64_trace));
}
#endif
