// Long-chain fold for d = 16, 32, 64 complex64 on tcgen05: the R- and S-passes of the reduce-
// then-scan in scan_long.cu (same tree, same carry contract) with every combine P <- A_t (x) P
// on the tensor cores instead of a lane group's FP32 FMAs.
//
// 128 / D chains share one CTA and one MMA (block-diagonal): A = [leaves of the chains,
// stacked] (128 x D), B = [states side by side] (D x 128), D_acc = A B (128 x 128 FP32 in TMEM,
// 3xTF32 like lmme_tc.cu); the 128 / D diagonal D x D blocks are the new states, the cross
// blocks are dropped (the step is latency- and shared-memory-bound, not tensor-bound). Per
// step:
//   warp 0      TMA: the next leaves (raw complex64, D / 16 K-blocks of [D rows x 16 k] per
//               chain) into the other A buffer (double-buffered);
//   warps 2-9   leaf transform in place: clamped row scale a_i = max(rowmax, 0) (Eq. 11,
//               core.py:252-253), sign * exp(x - a_i) -> (big, small) TF32 planes in the
//               64B-swizzled K-major layout (the same as lmme_tc.cu's A operand);
//   warp 1      D / 16 K-blocks x 2 x (small*big + big*small + big*big) MMAs, commit;
//   warps 10-13 epilogue, thread = state row i of chain h = i / D: the accumulator row's D
//               diagonal columns; output log = (log|acc| + a_i) + Q_h (the LMME epilogue
//               order, core.py:259) and sign; next right operand B_kj = U_j g_i with
//               U = acc 2^-e_i (exact; e_i the row maximum's binary exponent) and
//               g_i = exp((Q_h - Q'_h) + a_i + e_i ln2) <= 2 (the difference of the two state
//               scales first: no rounding at the magnitude of the chain's logs), Q'_h =
//               max(max_i log max_j |x_ij|, 0) the clamped maximum over the whole new state:
//               the right operand's scale is one value per state (the tile-scaled engine's
//               per-block scale, lmme_ts.cu), not per column — a state column more than ~e^87
//               below the state's largest entry flushes, as there. The B rows are written
//               K-major (one 4-byte word per (k, n); lanes 16-31 take the columns pair-swapped:
//               conflict-free).
// Prefixes (S-pass) or chain totals (R-pass) leave through a swizzled staging buffer per
// epilogue warp and TMA stores. A chain without a carry starts from its first leaf (raw,
// canonical signs), exactly as scan_long.cu. D <= 32 runs two CTAs per SM (smaller rings,
// a 2 KB staging box per warp, <= 72 registers).
#include "tc_ptx.cuh"

namespace goom {

namespace {
using namespace tc;

constexpr int kXW = 8;                               // leaf-transform warps
constexpr int kEW = 4;                               // epilogue warps (one per TMEM quadrant)
constexpr int kThreads = 64 + (kXW + kEW) * 32;      // 448
constexpr int kKB = 16384;                           // one K-block of A or B: 16 groups x 1 KB

template <int D>
struct FoldCfg {
  static_assert(D == 16 || D == 32 || D == 64, "tile-resident fold: D in {16, 32, 64}");
  static constexpr int kCPT = 128 / D;               // chains per tile
  static constexpr int kNKB = D / 16;                // K-blocks
  static constexpr int kAbuf = kNKB * kKB;           // the tile's leaves (A planes)
  static constexpr int kBoff = 2 * kAbuf;            // B planes (one buffer)
  static constexpr int kOutOff = kBoff + kNKB * kKB;
  // staging per epilogue warp: D = 64 two 128B-swizzled [32 x 16] boxes; else one
  // 64B-swizzled [32 x 8] box (fits two CTAs per SM)
  static constexpr int kBoxC = D == 64 ? 16 : 8;     // columns per box
  static constexpr int kBoxes = D == 64 ? 2 : 1;     // boxes per round
  static constexpr int kWarpOut = 32 * kBoxC * 8 * kBoxes;
  static constexpr int kRows = D < 32 ? D : 32;      // rows per box (one chain's rows in a warp)
  static constexpr int kRsOff = kOutOff + kEW * kWarpOut;  // leaf row scales [2][128]
  static constexpr int kQxOff = kRsOff + 2 * 128 * 4;      // D = 64: maxima [2 parities][4 warps]
  static constexpr int kBarOff = kQxOff + 64;
  static constexpr int kSmem = kBarOff + 128 + 1024;       // + barriers, + 1 KB alignment slack
  static constexpr int kMinBlocks = D == 64 ? 1 : 2;
  static_assert(kSmem * kMinBlocks <= 232448, "shared memory budget");
};

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
  const float2* A;        // leaves (T, D, D)
  int64_t T, s;           // chain k: leaves [k s, min(k s + s, T))
  const float2* carry0;   // chain 0's right carry (null: start from its first leaf)
  const float2* carries;  // chain k >= 1: carries[k - 1] (null: first leaf)
  float2* out;            // every prefix (S-pass) or null
  float2* tot;            // every chain's last state (R-pass) or null
  int64_t nchains;
};

// per chain of a tile: where it starts and how many combines it runs
struct ChainAt {
  int64_t t0, t1;   // leaves [t0, t1)
  const float2* cin;
  bool live;        // the chain exists
  __device__ __forceinline__ int64_t first() const { return cin ? t0 : t0 + 1; }
  __device__ __forceinline__ int64_t steps() const { return live ? t1 - first() : 0; }
};
__device__ __forceinline__ ChainAt chain_at(const FoldArgs& a, int64_t c, int d) {
  ChainAt r;
  r.live = c < a.nchains;
  r.t0 = c * a.s;
  r.t1 = r.t0 + a.s < a.T ? r.t0 + a.s : a.T;
  r.cin = !r.live ? nullptr
                  : (c == 0 ? a.carry0 : (a.carries ? a.carries + (c - 1) * d * d : nullptr));
  return r;
}

template <int D>
__global__ void __launch_bounds__(kThreads, FoldCfg<D>::kMinBlocks)
    long_fold_tc_kernel(const __grid_constant__ CUtensorMap mapA,
                        const __grid_constant__ CUtensorMap mapO, FoldArgs fa, int64_t ntiles) {
  using G = FoldCfg<D>;
  constexpr int kCPT = G::kCPT, kNKB = G::kNKB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t base = smem_u32(smem);
  float* rS = reinterpret_cast<float*>(smem + G::kRsOff);    // [buf][128]
  float* Qx = reinterpret_cast<float*>(smem + G::kQxOff);    // [parity][4 warps]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + G::kBarOff);
  uint64_t* a_full = bars;        // [2] leaves landed (tx bytes)
  uint64_t* a_ready = bars + 2;   // [2] leaves transformed (8 warps)
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
  // the tile's combine count: its longest chain
  auto tile_steps = [&](int64_t p) {
    int64_t n = 0;
#pragma unroll
    for (int h = 0; h < kCPT; ++h) n = max(n, chain_at(fa, kCPT * p + h, D).steps());
    return n;
  };

  if (warp == 0) {
    // ------------------------------ loader ------------------------------
    if (lane == 0) {
      int64_t g = 0;  // global step (A buffer g & 1)
      for (int64_t p = blockIdx.x; p < ntiles; p += gridDim.x) {
        const int64_t n = tile_steps(p);
        for (int64_t j = 0; j < n; ++j, ++g) {
          const int buf = (int)(g & 1);
          if (g >= 2) mbar_wait(smem_u32(&a_free[buf]), (uint32_t)(((g >> 1) - 1) & 1));
          uint32_t nvalid = 0;
#pragma unroll
          for (int h = 0; h < kCPT; ++h) nvalid += j < chain_at(fa, kCPT * p + h, D).steps() ? 1 : 0;
          const uint32_t bar = smem_u32(&a_full[buf]);
          mbar_expect_tx(bar, nvalid * (uint32_t)(D * D * 8));
          const uint32_t dst = base + (uint32_t)buf * G::kAbuf;
#pragma unroll
          for (int h = 0; h < kCPT; ++h) {  // chain h's rows: groups h D / 8 .. of each K-block
            const ChainAt c = chain_at(fa, kCPT * p + h, D);
            if (j >= c.steps()) continue;
            const int leaf = (int)(c.first() + j);
#pragma unroll
            for (int kb = 0; kb < kNKB; ++kb)
              tma_load_3d(dst + kb * kKB + h * D * 128, &mapA, kb * 16, 0, leaf, bar);
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
      for (int64_t p = blockIdx.x; p < ntiles; p += gridDim.x) {
        const int64_t n = tile_steps(p);
        for (int64_t j = 0; j < n; ++j, ++g, ++bw) {
          const int buf = (int)(g & 1);
          mbar_wait(smem_u32(&a_ready[buf]), (uint32_t)((g >> 1) & 1));
          L64_TRACE(0, g, clock64());
          mbar_wait(smem_u32(b_ready), (uint32_t)(bw & 1));
          tc_fence_after();
          L64_TRACE(1, g, clock64());
#pragma unroll
          for (int kb = 0; kb < kNKB; ++kb) {
            const uint32_t sa = base + (uint32_t)buf * G::kAbuf + kb * kKB;
            const uint32_t sb = base + G::kBoff + kb * kKB;
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
    // warp w: rows 16 w .. 16 w + 15 (one chain's) = groups 2w, 2w + 1 of every K-block;
    // lane: rows (lane >> 3) and 4 + (lane >> 3) of each group, k-pair lane & 7
    const int w = warp - 2, r = lane >> 3, kp = lane & 7;
    const int h = (16 * w) / D;  // chain of these rows
    int64_t g = 0;
    for (int64_t p = blockIdx.x; p < ntiles; p += gridDim.x) {
      const int64_t n = tile_steps(p);
      const int64_t mysteps = chain_at(fa, kCPT * p + h, D).steps();
      for (int64_t j = 0; j < n; ++j, ++g) {
        const int buf = (int)(g & 1);
        const uint32_t ab = base + (uint32_t)buf * G::kAbuf;
        mbar_wait(smem_u32(&a_full[buf]), (uint32_t)((g >> 1) & 1));
        if (w == 0 && lane == 0) L64_TRACE(6, g, clock64());
        const bool valid = j < mysteps;
        // the epilogue of step g - 2 has read this buffer's row scales
        if (g >= 2) mbar_wait(smem_u32(&rs_free[buf]), (uint32_t)(((g >> 1) - 1) & 1));
#pragma unroll
        for (int gg = 0; gg < 2; ++gg) {  // group 2w + gg: its 8 rows x D k held in registers
          float4 raw[2 * kNKB];           // [kb][a0 | a1]: one shared-memory read per element
          float s0 = 0.f, s1 = 0.f;       // rows r, r + 4
          bool odd = false;
          if (valid) {
            s0 = s1 = kNegInf;
#pragma unroll
            for (int kb = 0; kb < kNKB; ++kb) {
              const uint32_t ga = ab + kb * kKB + (2 * w + gg) * kGroupBytes;
              raw[2 * kb] = ld_shared_v4(ga + lane * 16);
              raw[2 * kb + 1] = ld_shared_v4(ga + 512 + lane * 16);
              s0 = fmaxf(s0, fmaxf(raw[2 * kb].x, raw[2 * kb].z));
              s1 = fmaxf(s1, fmaxf(raw[2 * kb + 1].x, raw[2 * kb + 1].z));
              odd |= odd_phase(raw[2 * kb].y) | odd_phase(raw[2 * kb].w) |
                     odd_phase(raw[2 * kb + 1].y) | odd_phase(raw[2 * kb + 1].w);
            }
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
              s0 = fmaxf(s0, __shfl_xor_sync(0xffffffffu, s0, o));
              s1 = fmaxf(s1, __shfl_xor_sync(0xffffffffu, s1, o));
            }
            s0 = fmaxf(s0, 0.0f);  // Eq. 11 clamp
            s1 = fmaxf(s1, 0.0f);
          }
          const bool canon = !__any_sync(0xffffffffu, odd);  // phases all 0 / pi: cheap sign
          if (kp == 0) {
            rS[buf * 128 + 16 * w + 8 * gg + r] = s0;
            rS[buf * 128 + 16 * w + 8 * gg + r + 4] = s1;
          }
          __syncwarp();  // the group is in registers before it is overwritten
#pragma unroll
          for (int kb = 0; kb < kNKB; ++kb) {
            const uint32_t ga = ab + kb * kKB + (2 * w + gg) * kGroupBytes;
            uint32_t hb[4], lb[4];
            if (valid) {
              const float4 a0 = raw[2 * kb], a1 = raw[2 * kb + 1];
              if (canon) {
                goom_split<true>(make_float2(a0.x, a0.y), s0, hb[0], lb[0]);
                goom_split<true>(make_float2(a0.z, a0.w), s0, hb[1], lb[1]);
                goom_split<true>(make_float2(a1.x, a1.y), s1, hb[2], lb[2]);
                goom_split<true>(make_float2(a1.z, a1.w), s1, hb[3], lb[3]);
              } else {
                goom_split<false>(make_float2(a0.x, a0.y), s0, hb[0], lb[0]);
                goom_split<false>(make_float2(a0.z, a0.w), s0, hb[1], lb[1]);
                goom_split<false>(make_float2(a1.x, a1.y), s1, hb[2], lb[2]);
                goom_split<false>(make_float2(a1.z, a1.w), s1, hb[3], lb[3]);
              }
            } else {  // a finished chain multiplies by the identity (its output is dropped)
              const int row = (16 * w + 8 * gg + r) % D, k0 = kb * 16 + 2 * kp;
              hb[0] = row == k0 ? 0x3f800000u : 0u;
              hb[1] = row == k0 + 1 ? 0x3f800000u : 0u;
              hb[2] = row + 4 == k0 ? 0x3f800000u : 0u;
              hb[3] = row + 4 == k0 + 1 ? 0x3f800000u : 0u;
              lb[0] = lb[1] = lb[2] = lb[3] = 0u;
            }
            const uint32_t o0 = sw64_off(r, kp >> 1) + (kp & 1) * 8;
            const uint32_t o1 = sw64_off(r + 4, kp >> 1) + (kp & 1) * 8;
            st_shared_v2(ga + o0, hb[0], hb[1]);
            st_shared_v2(ga + 512 + o0, lb[0], lb[1]);
            st_shared_v2(ga + o1, hb[2], hb[3]);
            st_shared_v2(ga + 512 + o1, lb[2], lb[3]);
          }
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
    const int h = i / D, k = i % D;                    // chain, state row
    const int hw = D == 64 ? (quad & 1) : 0;           // D = 64: this warp's half of the chain
    const uint32_t stage = base + G::kOutOff + (uint32_t)e * G::kWarpOut;
    const uint32_t bplane = base + G::kBoff;
    int64_t g = 0, par = 0;  // global step; reduction parity
    // chain max of v over its D rows, clamped at 0 (D = 64: two warps, a named barrier)
    auto chain_max = [&](float v) {
      if constexpr (D == 64) {
        v = warp_max(v);
        if (lane == 0) Qx[(par & 1) * 4 + quad] = v;
        asm volatile("bar.sync %0, 64;" ::"r"(1 + h) : "memory");
        v = fmaxf(Qx[(par & 1) * 4 + 2 * h], Qx[(par & 1) * 4 + 2 * h + 1]);
        ++par;
      } else {
#pragma unroll
        for (int o = D / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
      }
      return fmaxf(v, 0.0f);
    };
    // this thread's state row as the next right operand: B[k][D h + n] = f(n) (lanes 16-31
    // take the columns in pair-swapped order: their rows share banks with lanes 0-15's)
    auto write_b = [&](auto f) {
#pragma unroll
      for (int jj = 0; jj < D; ++jj) {
        const bool sw = lane >= 16;
        const float x = sw ? f(jj ^ 1) : f(jj);
        const uint32_t big = tf32_round(x), small = __float_as_uint(x - __uint_as_float(big));
        const uint32_t off = kmaj_off(k, D * h + (jj ^ (sw ? 1 : 0)));
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(bplane + off), "r"(big) : "memory");
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(bplane + off + 512), "r"(small) : "memory");
      }
    };
    // stage the warp's rows (o(n): complex64 of column n of this thread's row) and TMA-store
    // them: rounds of kBoxes boxes of kBoxC columns; a box holds one chain's kRows rows
    // (D = 16: two chains per warp, matrices mat0 / mat1; a chain with ok* false is skipped)
    auto store_rows = [&](auto o, int64_t mat0, bool ok0, int64_t mat1, bool ok1) {
      constexpr int kC = G::kBoxC, kRb = kC * 8;  // columns per box, bytes per staged row
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += kC * G::kBoxes) {
        if (lane == 0) tma_store_wait_read<0>();
        __syncwarp();
#pragma unroll
        for (int bx = 0; bx < G::kBoxes; ++bx)
#pragma unroll
          for (int c = 0; c < kC / 2; ++c) {  // 16-byte chunk c of this row
            const float2 p0 = o(c0 + bx * kC + 2 * c), p1 = o(c0 + bx * kC + 2 * c + 1);
            const int cs = kC == 16 ? (c ^ (lane & 7)) : (c ^ ((lane >> 1) & 3));  // 128B / 64B
            st_shared_v4(stage + bx * 32 * kRb + lane * kRb + (cs << 4), __float_as_uint(p0.x),
                         __float_as_uint(p0.y), __float_as_uint(p1.x), __float_as_uint(p1.y));
          }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int bx = 0; bx < G::kBoxes; ++bx) {
            if (ok0)
              tma_store_3d(&mapO, stage + bx * 32 * kRb, c0 + bx * kC, 32 * hw, (int)mat0);
            if (D == 16 && ok1)
              tma_store_3d(&mapO, stage + bx * 32 * kRb + 16 * kRb, c0 + bx * kC, 0, (int)mat1);
          }
        }
        __syncwarp();
      }
    };
    // a row of D complex64 straight to global (once per chain: raw first leaves, totals)
    auto put_row = [&](float2* dst, auto o) {
      float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
      for (int q = 0; q < D / 2; ++q) {
        const float2 a0 = o(2 * q), a1 = o(2 * q + 1);
        d4[q] = make_float4(a0.x, a0.y, a1.x, a1.y);
      }
    };
    for (int64_t p = blockIdx.x; p < ntiles; p += gridDim.x) {
      const ChainAt cm = chain_at(fa, kCPT * p + h, D);
      // D = 16: the warp's two chains (rows 0-15, 16-31) for the TMA stores
      const ChainAt cw0 = chain_at(fa, kCPT * p + (32 * quad) / D, D);
      const ChainAt cw1 = chain_at(fa, kCPT * p + (32 * quad + 16) / D, D);
      const int64_t n = tile_steps(p);
      const int64_t mysteps = cm.steps();
      // initial state: the carry, or the chain's first leaf (raw), or the identity for a
      // chain that does not exist; Q = its clamped maximum log
      float Q;
      {
        const float2* src = cm.live ? (cm.cin ? cm.cin : fa.A + cm.t0 * D * D) : nullptr;
        const float2* srow = src ? src + k * D : nullptr;
        float m = kNegInf;
        if (srow) {
#pragma unroll 8
          for (int q = 0; q < D; ++q) m = fmaxf(m, __ldg(&srow[q].x));
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
          if (fa.out) put_row(fa.out + cm.t0 * D * D + k * D, rawc);
          if (fa.tot && cm.t1 - cm.t0 == 1) put_row(fa.tot + (kCPT * p + h) * D * D + k * D, rawc);
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
        uint32_t acc[D];
        if constexpr (D == 16) {
          // tcgen05.ld is warp-collective (one column range for all lanes): the warp's two
          // chains' diagonal blocks are columns 32 quad .. + 15 (lanes 0-15) and + 16 .. + 31
          uint32_t v[32];
          tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(32 * quad), v);
#pragma unroll
          for (int q = 0; q < 16; ++q) acc[q] = lane < 16 ? v[q] : v[q + 16];
        } else {
#pragma unroll
          for (int q = 0; q < D; q += 32)
            tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(D * h + q),
                      *reinterpret_cast<uint32_t(*)[32]>(&acc[q]));
        }
        const bool valid = j < mysteps;
        const bool more = j + 1 < n;
        // new state: row maximum, its binary exponent, the clamped chain maximum log
        float m = 0.0f;
#pragma unroll
        for (int q = 0; q < D; ++q) m = fmaxf(m, fabsf(__uint_as_float(acc[q])));
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
        if (fa.out) {
          const bool ok0 = j < cw0.steps(), ok1 = j < cw1.steps();
          if (__any_sync(0xffffffffu, valid))
            store_rows(outc, cw0.first() + j, ok0, cw1.first() + j, ok1);
        }
        if (valid && fa.tot && j + 1 == mysteps) put_row(fa.tot + (kCPT * p + h) * D * D + k * D, outc);
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

template <int D>
int launch_fold_tc_d(const float2* A, int64_t T, int64_t s, const float2* carry0,
                     const float2* carries, float2* out, float2* tot, cudaStream_t st) {
  using G = FoldCfg<D>;
  GOOM_TRY(smem_attr((const void*)long_fold_tc_kernel<D>, G::kSmem, "long_fold_tc smem"));
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (out && (reinterpret_cast<uintptr_t>(out) & 15)) ||
      (tot && (reinterpret_cast<uintptr_t>(tot) & 15)))
    return fail(GOOM_EUNSUPPORTED, "long_fold_tc: 16-byte aligned tensors");
  alignas(64) CUtensorMap mapA, mapO;
  {  // leaves (k, row, matrix) complex64 as int64, box 16 k x D rows
    cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)D, (cuuint64_t)T};
    cuuint64_t strides[2] = {(cuuint64_t)D * 8, (cuuint64_t)D * D * 8};
    cuuint32_t box[3] = {16, (cuuint32_t)D, 1};
    GOOM_TRY(encode(&mapA, Operand{A, 0, 1}, 3, dims, strides, box));
  }
  if (out) {  // prefixes (col, row, matrix), box kBoxC cols x kRows rows (128B / 64B swizzle)
    cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)D, (cuuint64_t)T};
    cuuint64_t strides[2] = {(cuuint64_t)D * 8, (cuuint64_t)D * D * 8};
    cuuint32_t box[3] = {(cuuint32_t)G::kBoxC, (cuuint32_t)G::kRows, 1};
    GOOM_TRY(encode(&mapO, Operand{out, 0, 1}, 3, dims, strides, box,
                    G::kBoxC == 16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B));
  } else {
    mapO = mapA;  // unused
  }
  FoldArgs fa{A, T, s, carry0, carries, out, tot, (T + s - 1) / s};
  const int64_t ntiles = (fa.nchains + G::kCPT - 1) / G::kCPT;
  const int64_t slots = (int64_t)num_sms() * G::kMinBlocks;
  const unsigned grid = (unsigned)(ntiles < slots ? ntiles : slots);
  long_fold_tc_kernel<D><<<grid, kThreads, G::kSmem, st>>>(mapA, mapO, fa, ntiles);
  GOOM_CHECK_LAUNCH("long_fold_tc_kernel");
  return GOOM_OK;
}

}  // namespace

// d = 16 / 32 / 64 complex64: the tile-resident fold (see the header comment)
bool fold_tc_eligible(int d) { return d == 16 || d == 32 || d == 64; }

int launch_fold_tc(const float2* A, int64_t T, int d, int64_t s, const float2* carry0,
                   const float2* carries, float2* out, float2* tot, cudaStream_t st) {
  if (d == 16) return launch_fold_tc_d<16>(A, T, s, carry0, carries, out, tot, st);
  if (d == 32) return launch_fold_tc_d<32>(A, T, s, carry0, carries, out, tot, st);
  if (d == 64) return launch_fold_tc_d<64>(A, T, s, carry0, carries, out, tot, st);
  return fail(GOOM_EUNSUPPORTED, "tile-resident fold: d in {16, 32, 64}");
}

}  // namespace goom

#ifdef GOOM_L64_TRACE
extern "C" int goom_l64_trace_read(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, goom::g_l64_trace, sizeof(goom::g_l64_trace));
}
#endif
