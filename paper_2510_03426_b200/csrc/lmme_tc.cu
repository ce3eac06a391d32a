// tcgen05 LMME for complex64 GOOMs: Eq. 10-12 with the real GEMM on the 5th-gen
// tensor cores at FP32 accuracy (3xTF32), everything else fused around it.
//
// Persistent kernel: one CTA per SM walks 128 x BN output tiles (BN = 256, or 128 when
// m % 256 != 0; full K per tile). A STAGES-deep ring of 16-wide K-blocks, each stage used
// twice in place, and a double-buffered TMEM accumulator so the epilogue of tile i
// overlaps the main loop of tile i+1:
//   warp 0        loader   : TMA (cp.async.bulk.tensor) of the raw complex64 K-block:
//                            A as 16 groups of 8 rows x 16 k, B as BN/8 groups of
//                            16 k x 8 columns; every group is 1 KB of complex64;
//   warps 2..17   transform: each warp owns whole groups; it reads a group into
//                            registers, v = sign * exp(log - scale) (clamped scales from
//                            the pre-pass or the producing epilogue), splits v = big +
//                            small (TF32, round to nearest) and writes the two 512 B TF32
//                            planes of the group back into the SAME 1 KB, in the
//                            64B-swizzled K-major layout the UMMA descriptors read
//                            (SBO = 1 KB, big and small planes interleaved per group).
//                            No real matrix ever touches HBM and no second ring is needed;
//   warp 1        MMA      : one thread issues per 8-wide K step three
//                            tcgen05.mma.cta_group::1.kind::tf32 into the tile's TMEM
//                            accumulator: small*big + big*small + big*big;
//   warps 18..    epilogue : tcgen05.ld the accumulator, (log|I| + a_i) + b_j and the
//                            sign in registers (log via lg2.approx: abs. error ~1e-7,
//                            below the FP32 ulp of the output), optional fused gadd,
//                            store, and optionally the clamped row / column maxima of the
//                            output (the next LMME's scales: no pre-pass over C). BN = 128:
//                            8 warps (two per TMEM lane quadrant, 64 columns each); BN = 256: 4.
//
// kFuse (no scales given, BN = 128): Eq. 11's clamped scales (core.py:252-253) come from a
// SCALE PASS through the same ring instead of the row / column pre-pass. The loader issues
// every K-block of a tile twice: once one tile AHEAD (scale stage) and once for the main
// loop, interleaved [main(t, kb), scale(t + 1, kb)], so the HBM read of tile t+1 overlaps the
// L2 re-read + MMA of tile t. A transform warp reduces, from the scale stages, the maxima of
// exactly the A rows and B columns it later transforms (its own groups), so the scales never
// cross warps on the way to the transform; the warp publishes them to a 4-slot table for the
// epilogue. Its phase check ("all phases 0 / pi" fast path) is per warp as well. Max is
// order-independent, so the scales are bitwise the pre-pass's.
//
// Error budget: plain TF32 gives ~3e-4 Frobenius error at d = 1024;
// 3xTF32 keeps the single-LMME Frobenius error below 1e-5 up to k = 1024 (the
// tensor core's FP32 accumulation, not the split, sets the floor; measured
// in tools/precision_probe.py).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "tc_ptx.cuh"

namespace goom {

namespace {
using namespace tc;

constexpr int BM = 128;
constexpr int BK = 16;        // K per stage: 16 TF32 = one 64-byte swizzle row
constexpr int kXformWarps = 16;
constexpr int kGroupBytes = 1024;                // 8 rows x 16 k complex64 == 2 x 512 B TF32
constexpr int kScaleSlots = 4;                   // kFuse: per-tile scale tables (epilogue)

template <int BN, bool kFuse>
struct Cfg {
  static constexpr int kEpiWarps = BN == 128 ? 8 : 4;  // 2 / 1 per TMEM lane quadrant
  static constexpr int kEpiCols = BN / (kEpiWarps / 4);  // accumulator columns per warp
  static constexpr int kThreads = 64 + (kXformWarps + kEpiWarps) * 32;
  static constexpr int kStages = BN == 128 ? 6 : 4;      // ring depth
  static constexpr int kStageOut = BN == 128 ? 2048 : 8192;  // staging per warp: 32 rows x 8 / 32 cols
  static constexpr bool kTmaOut = BN == 128;  // staging stored by TMA (64B-swizzled box)
  static constexpr int kGroupsA = BM / 8;
  static constexpr int kGroupsB = BN / 8;
  static constexpr int kBytesA = kGroupsA * kGroupBytes;
  static constexpr int kStage = (kGroupsA + kGroupsB) * kGroupBytes;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered FP32 accumulator
  static constexpr int kRing = kStages * kStage;
  static constexpr int kBars = 1024;        // mbarriers + TMEM slot (keeps the staging 1 KB-aligned)
  static constexpr int kOut = kRing + kBars;  // epilogue staging: [warp][32 rows][16 / 32 cols]
  static constexpr int kScaleOff = kOut + kEpiWarps * kStageOut;
  static constexpr int kScaleBytes = kFuse ? kScaleSlots * (BM + BN) * 4 : 0;
  static constexpr int kSmem = kScaleOff + kScaleBytes + 1024;
};

// (PTX helpers: tc_ptx.cuh)

// Transform of one stage, in place (see the header comment), split in two halves so the
// raw loads of stage g+1 are in flight while stage g is transformed (software pipeline).
// A group (raw [8 rows][16 k]): lane l holds 16 B (k-pair) at l*16 and 512 + l*16 -> rows
// l/8 and 4 + l/8, k-pair l%8 (conflict-free); it writes its 2 TF32 of each row as 8-byte
// halves of the swizzled chunk. B group (raw [16 k][8 cols]): lane (n = l%8, c = l/8)
// gathers k = 4c..4c+3 of column n. Each transform warp owns A group xw and B groups
// xw (+ 16): the same groups for every stage, so its scales live in registers.
template <int NB>
struct RawStage {
  static constexpr int kB = NB / kXformWarps;  // B groups per warp (1 or 2)
  float4 a0, a1;
  float2 b[kB][4];
};

template <int NB>
__device__ __forceinline__ void load_stage(uint32_t base, int xw, int lane, RawStage<NB>& raw) {
  const uint32_t ga = base + xw * kGroupBytes;
  raw.a0 = ld_shared_v4(ga + lane * 16);
  raw.a1 = ld_shared_v4(ga + 512 + lane * 16);
  const int bn = lane & 7, bc = lane >> 3;
#pragma unroll
  for (int i = 0; i < RawStage<NB>::kB; ++i) {
    const uint32_t gb = base + (BM / 8 + xw + i * kXformWarps) * kGroupBytes;
#pragma unroll
    for (int j = 0; j < 4; ++j) raw.b[i][j] = ld_shared_v2(gb + (4 * bc + j) * 64 + bn * 8);
  }
}

template <int NB>
__device__ __forceinline__ void load_stage_b(uint32_t base, int xw, int lane, RawStage<NB>& raw) {
  const int bn = lane & 7, bc = lane >> 3;
#pragma unroll
  for (int i = 0; i < RawStage<NB>::kB; ++i) {
    const uint32_t gb = base + (BM / 8 + xw + i * kXformWarps) * kGroupBytes;
#pragma unroll
    for (int j = 0; j < 4; ++j) raw.b[i][j] = ld_shared_v2(gb + (4 * bc + j) * 64 + bn * 8);
  }
}

template <int NB, bool kCanon>
__device__ __forceinline__ void store_stage(uint32_t base, int xw, int lane,
                                            const RawStage<NB>& raw, float sa0, float sa1,
                                            const float (&sb)[2]) {
  const int r = lane >> 3, kp = lane & 7;
  uint32_t ha[4], la[4];
  goom_split<kCanon>(make_float2(raw.a0.x, raw.a0.y), sa0, ha[0], la[0]);
  goom_split<kCanon>(make_float2(raw.a0.z, raw.a0.w), sa0, ha[1], la[1]);
  goom_split<kCanon>(make_float2(raw.a1.x, raw.a1.y), sa1, ha[2], la[2]);
  goom_split<kCanon>(make_float2(raw.a1.z, raw.a1.w), sa1, ha[3], la[3]);
  uint32_t hb[RawStage<NB>::kB][4], lb[RawStage<NB>::kB][4];
#pragma unroll
  for (int i = 0; i < RawStage<NB>::kB; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) goom_split<kCanon>(raw.b[i][j], sb[i], hb[i][j], lb[i][j]);
  __syncwarp();  // every lane's groups are in registers before any is overwritten
  const uint32_t ga = base + xw * kGroupBytes;
  const uint32_t o0 = sw64_off(r, kp >> 1) + (kp & 1) * 8;
  const uint32_t o1 = sw64_off(r + 4, kp >> 1) + (kp & 1) * 8;
  st_shared_v2(ga + o0, ha[0], ha[1]);
  st_shared_v2(ga + 512 + o0, la[0], la[1]);
  st_shared_v2(ga + o1, ha[2], ha[3]);
  st_shared_v2(ga + 512 + o1, la[2], la[3]);
  const int bn = lane & 7, bc = lane >> 3;
  const uint32_t ob = sw64_off(bn, bc);
#pragma unroll
  for (int i = 0; i < RawStage<NB>::kB; ++i) {
    const uint32_t gb = base + (BM / 8 + xw + i * kXformWarps) * kGroupBytes;
    st_shared_v4(gb + ob, hb[i][0], hb[i][1], hb[i][2], hb[i][3]);
    st_shared_v4(gb + 512 + ob, lb[i][0], lb[i][1], lb[i][2], lb[i][3]);
  }
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

struct TileGrid {
  int nct, nrt;       // column / row tiles per product
  int64_t b_base;     // first product of this launch
  int64_t tiles;      // tiles in this launch
  int64_t batch;      // kDuo: products (a tile holds products 2t, 2t + 1)
  __device__ __forceinline__ void at(int64_t t, int64_t& b, int& row0, int& col0, int BN) const {
    const int ct = (int)(t % nct);
    const int64_t q = t / nct;
    row0 = (int)(q % nrt) * BM;
    col0 = ct * BN;
    b = b_base + q / nrt;
  }
};

#ifdef GOOM_TC_TRACE
// profiling build only (tools/tc_trace.py): clock64 stamps of CTA 0's ring positions
__device__ long long g_tc_trace[8][256];
#define TC_TRACE(row, i, v) \
  do {                          \
    if (blockIdx.x == 0 && (i) < 256) g_tc_trace[row][i] = (v); \
  } while (0)
#else
#define TC_TRACE(row, i, v) \
  do {                        \
  } while (0)
#endif

struct Emit {
  float* row;   // row[b * row_stride + i]: clamped row maxima of C (atomicMax on the bits)
  int64_t row_stride;
  float* col;   // col[b * col_stride + j]
  int64_t col_stride;
};

// Persistent kernel: grid = min(tiles, SMs); tiles in row-major (product, row tile, column
// tile) order, so concurrently resident tiles share operand panels in L2.
template <int BN, bool kFuse, bool kDuo>
__global__ void __launch_bounds__(Cfg<BN, kFuse>::kThreads, 1)
    lmme_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ CUtensorMap mapB3, const __grid_constant__ CUtensorMap mapC,
                   Operand A, Operand B, Operand D, Scales rowA, Scales colB,
                   float2* __restrict__ C, int64_t strideC, TileGrid grid, int n, int k, int m,
                   const int* __restrict__ noncanon, Emit emit, int debug) {
  using G = Cfg<BN, kFuse>;
  constexpr int kEpiWarps = G::kEpiWarps;
  constexpr int STAGES = G::kStages;
  const int pf = (debug >> 8) & 15;  // kFuse: L2 prefetch distance (GOOM_TC_PREFETCH)
  const int fflags = debug & 0xF0;  // kFuse probes: 16 A row chunks, 32 no L2 hints, 64 late
  // FuseSeq lateness: GOOM_TC1_LATE (default 1), or 2 with GOOM_TC_DEBUG bit 64
  const int late = (fflags & 64) ? 2 : ((debug >> 12) & 15);
  debug &= 15;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KB-align the ring while keeping the pointer's shared-space provenance
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + G::kRing);
  uint64_t* full = bars;                    // [STAGES] TMA landed (tx bytes)
  uint64_t* ready = bars + STAGES;          // [STAGES] operands transformed (16 warp arrivals)
  uint64_t* freed = bars + 2 * STAGES;      // [STAGES] MMAs of the stage retired (commit)
  uint64_t* sfreed = bars + 3 * STAGES;     // [STAGES] kFuse: scale stage read (16 warps)
  uint64_t* acc_full = bars + 4 * STAGES;   // [2] accumulator buffer complete (commit)
  uint64_t* acc_empty = acc_full + 2;       // [2] epilogue drained the buffer
  uint64_t* sc_full = acc_empty + 2;        // [kScaleSlots] kFuse: a tile's scale tables
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sc_full + kScaleSlots);
  float* rowS = reinterpret_cast<float*>(smem + G::kScaleOff);  // kFuse [slot][BM]
  float* colS = rowS + kScaleSlots * BM;                         // kFuse [slot][BN]

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nk = k / BK;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&ready[s]), kXformWarps);
      mbar_init(smem_u32(&freed[s]), 1);
      mbar_init(smem_u32(&sfreed[s]), kXformWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&acc_full[i]), 1);
      mbar_init(smem_u32(&acc_empty[i]), kEpiWarps);
    }
    for (int i = 0; i < kScaleSlots; ++i) mbar_init(smem_u32(&sc_full[i]), kXformWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // the MMA warp owns the TMEM allocation: two BN-column accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(G::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t ring = smem_u32(smem);

  // kFuse scale stages: A as contiguous 16 KB row chunks (one bulk copy) instead of the
  // K-block box (GOOM_TC_DEBUG bit 16; k % 64 == 0) — measured slower, kept as a probe
  const bool rowsA = kFuse && (k % 64) == 0 && (fflags & 16) != 0;
  // kFuse L2 policy (GOOM_TC_DEBUG bit 32 off): scale-pass loads evict_last (the main pass
  // re-reads them one tile later), main-pass loads evict_first, output stores evict_first
  const bool hints = kFuse && (fflags & 32) == 0;
  const uint64_t pol_keep = policy_evict_last(), pol_drop = policy_evict_first();
  // a tile's load coordinates, computed once per tile (the loader is one thread: int64
  // divisions per stage measured ~1.5 k clocks per issue, slower than the ring drains)
  struct TileAt {
    int64_t t = -1;
    const float2* abase;  // the tile's 128 A rows (contiguous)
    int row0, col0, ma, mb;
    int ma1, mb1;  // kDuo: matrices of the tile's second product
  };
  auto tile_at = [&](int64_t t, TileAt& c) {
    if (c.t == t) return;
    c.t = t;
    if constexpr (kDuo) {  // products 2t and 2t + 1 (the last tile of an odd batch repeats 2t)
      const int64_t b = 2 * t, b1 = b + 1 < grid.batch ? b + 1 : b;
      c.row0 = c.col0 = 0;
      c.ma = A.stride == 0 ? 0 : (int)(b / A.div);
      c.mb = B.stride == 0 ? 0 : (int)(b / B.div);
      c.ma1 = A.stride == 0 ? 0 : (int)(b1 / A.div);
      c.mb1 = B.stride == 0 ? 0 : (int)(b1 / B.div);
      c.abase = A.ptr;
      return;
    }
    int64_t b;
    grid.at(t, b, c.row0, c.col0, BN);
    c.ma = A.stride == 0 ? 0 : (int)(b / A.div);
    c.mb = B.stride == 0 ? 0 : (int)(b / B.div);
    c.abase = A.at(b) + (int64_t)c.row0 * k;
  };
  // one K-block of a tile into ring slot s (scale stage: A rows as a contiguous chunk)
  auto issue_loads = [&](int s, const TileAt& c, int kb, bool scale) {
    const uint32_t bar = smem_u32(&full[s]);
    mbar_expect_tx(bar, G::kStage);
    const uint32_t dst = ring + s * G::kStage;
    const int k0 = kb * BK;
    if constexpr (kDuo) {
      // [product 0: 64 rows | product 1: 64 rows][16 k]; B groups 0-7 product 0, 8-15 product 1
      const uint64_t pol = scale ? pol_keep : pol_drop;
      tma_load_3d_hint(dst, &mapA, k0, 0, c.ma, bar, pol);
      tma_load_3d_hint(dst + G::kBytesA / 2, &mapA, k0, 0, c.ma1, bar, pol);
      tma_load_4d_hint(dst + G::kBytesA, &mapB, 0, k0, 0, c.mb, bar, pol);
      tma_load_4d_hint(dst + G::kBytesA + (G::kStage - G::kBytesA) / 2, &mapB, 0, k0, 0, c.mb1, bar,
                       pol);
      return;
    }
    if (scale && rowsA)  // float4 chunk kb of the tile's 128 contiguous A rows
      bulk_g2s(dst, c.abase + kb * (G::kBytesA / 8), G::kBytesA, bar);
    else if (hints)  // kFuse: the scale pass keeps its lines for the main pass, which frees them
      tma_load_3d_hint(dst, &mapA, k0, c.row0, c.ma, bar, scale ? pol_keep : pol_drop);
    else
      tma_load_3d(dst, &mapA, k0, c.row0, c.ma, bar);                      // [128 rows][16 k]
    if (debug == 6)  /* profiling aid: B as one 2 KB-row box (layout wrong) */
      tma_load_3d(dst + G::kBytesA, &mapB3, c.col0, k0, c.mb, bar);
    else if (hints)
      tma_load_4d_hint(dst + G::kBytesA, &mapB, 0, k0, c.col0 / 8, c.mb, bar,
                       scale ? pol_keep : pol_drop);
    else
      tma_load_4d(dst + G::kBytesA, &mapB, 0, k0, c.col0 / 8, c.mb, bar);  // [BN/8][16 k][8 cols]
  };

  if (warp == 0) {
    // ------------------------------ loader ------------------------------
    if (lane == 0) {
      if constexpr (kDuo) {
        // resident tiles: each K-block is loaded once; the transform reduces the scales from
        // the landed stages of the whole tile before it transforms any of them
        TileAt c;
        int64_t g = 0;
        for (int64_t t = blockIdx.x; t < grid.tiles; t += gridDim.x) {
          tile_at(t, c);
          for (int kb = 0; kb < nk; ++kb, ++g) {
            const int s = (int)(g % STAGES);
            mbar_wait(smem_u32(&freed[s]), (uint32_t)((g / STAGES) & 1) ^ 1u);
            issue_loads(s, c, kb, false);
          }
        }
      } else if constexpr (kFuse) {
        // L2 prefetch of a whole tile (A panel, and the B panel when it is contiguous) `pf`
        // tiles ahead of the main loop, so its scale stages hit L2 (GOOM_TC_PREFETCH)
        auto prefetch_tile = [&](int64_t tp) {
          if (tp >= grid.tiles) return;
          int64_t b;
          int row0, col0;
          grid.at(tp, b, row0, col0, BN);
          prefetch_l2(A.at(b) + (int64_t)row0 * k, (uint32_t)BM * (uint32_t)k * 8u);
          if (m == BN) prefetch_l2(B.at(b), (uint32_t)k * (uint32_t)m * 8u);
        };
        for (int i = 1; i < pf; ++i) prefetch_tile(blockIdx.x + (int64_t)i * gridDim.x);
        RingBits<STAGES> rb;
        int gpos = 0;
        TileAt cm, cs;  // coordinates of the main-pass and the scale-pass tile
        for (FuseSeq q(blockIdx.x, gridDim.x, grid.tiles, nk, late); q.valid(); q.next()) {
          const int s = rb.s;
          if (pf > 0 && !q.scale() && q.kb == 0) prefetch_tile(q.t + (int64_t)pf * q.step);
          if (rb.bit(rb.used)) {  // wait for the slot's previous occupant to be released
            if (rb.bit(rb.last_scale))
              mbar_wait(smem_u32(&sfreed[s]), rb.bit(rb.scalep) ^ 1u);
            else
              mbar_wait(smem_u32(&freed[s]), rb.bit(rb.mainp) ^ 1u);
          }
          TC_TRACE(0, gpos, clock64());
          TileAt& c = q.scale() ? cs : cm;
          tile_at(q.tile(), c);
          issue_loads(s, c, q.block(), q.scale());
          rb.advance(q.scale());
          ++gpos;
        }
      } else {
        int64_t g = 0;  // K-blocks issued so far (ring position)
        TileAt c;
        for (int64_t t = blockIdx.x; t < grid.tiles; t += gridDim.x) {
          tile_at(t, c);
          for (int kb = 0; kb < nk; ++kb, ++g) {
            const int s = (int)(g % STAGES);
            mbar_wait(smem_u32(&freed[s]), (uint32_t)((g / STAGES) & 1) ^ 1u);
            if (debug >= 3) {  // profiling aid: no loads
              mbar_arrive(smem_u32(&full[s]));
              continue;
            }
            issue_loads(s, c, kb, false);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ------------------------------
    if (lane == 0) {
      constexpr uint32_t idesc = tf32_idesc(BM, BN);
      auto mma_stage = [&](int s, int kb, uint32_t acc) {
        const uint32_t base = ring + s * G::kStage;
        const uint64_t dAb = sw64_desc(base), dAs = sw64_desc(base + 512);
        const uint64_t dBb = sw64_desc(base + G::kBytesA);
        const uint64_t dBs = sw64_desc(base + G::kBytesA + 512);
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint64_t adv = (uint64_t)(kk * 32) >> 4;  // 8 TF32 = 32 B along K
          mma_tf32(acc, dAs + adv, dBb + adv, idesc, (kb | kk) != 0);
          mma_tf32(acc, dAb + adv, dBs + adv, idesc, 1);
          mma_tf32(acc, dAb + adv, dBb + adv, idesc, 1);
        }
      };
      if constexpr (kFuse && !kDuo) {
        RingBits<STAGES> rb;
        int gpos = 0;
        int lt = -1;  // local tile counter -> accumulator buffer lt & 1
        uint32_t acc = tmem;
        for (FuseSeq q(blockIdx.x, gridDim.x, grid.tiles, nk, late); q.valid(); q.next()) {
          const int s = rb.s;
          const bool sc = q.scale();
          if (!sc) {
            if (q.kb == 0) {
              ++lt;
              mbar_wait(smem_u32(&acc_empty[lt & 1]), (uint32_t)((lt >> 1) & 1) ^ 1u);
              tc_fence_after();
              acc = tmem + (uint32_t)((lt & 1) * BN);
            }
            mbar_wait(smem_u32(&ready[s]), rb.bit(rb.mainp));
            tc_fence_after();
            TC_TRACE(3, gpos, clock64());
            mma_stage(s, q.kb, acc);
            mma_commit(smem_u32(&freed[s]));  // the stage returns to the loader
            if (q.kb == nk - 1) mma_commit(smem_u32(&acc_full[lt & 1]));
          }
          rb.advance(sc);
          ++gpos;
        }
      } else {
        int64_t g = 0;
        int lt = 0;  // local tile counter -> accumulator buffer lt & 1
        for (int64_t t = blockIdx.x; t < grid.tiles; t += gridDim.x, ++lt) {
          const int buf = lt & 1;
          mbar_wait(smem_u32(&acc_empty[buf]), (uint32_t)((lt >> 1) & 1) ^ 1u);
          tc_fence_after();
          const uint32_t acc = tmem + (uint32_t)(buf * BN);
          for (int kb = 0; kb < nk; ++kb, ++g) {
            const int s = (int)(g % STAGES);
            mbar_wait(smem_u32(&ready[s]), (uint32_t)((g / STAGES) & 1));
            tc_fence_after();
            if (debug != 2 && debug < 5) mma_stage(s, kb, acc);
            mma_commit(smem_u32(&freed[s]));  // the stage returns to the loader when these retire
          }
          mma_commit(smem_u32(&acc_full[buf]));  // accumulator of this tile complete
        }
      }
    }
    __syncwarp();
  } else if (warp < 2 + kXformWarps) {
    // ------------------------------ transform (in place, software-pipelined) ---------------
    const int xw = warp - 2;
    const int r = lane >> 3, bn = lane & 7;
    float sa0 = 0.f, sa1 = 0.f, sb[2] = {0.f, 0.f};
    if constexpr (kDuo) {
      // resident tiles (k = 64: a tile's 4 K-blocks fit the ring): wait for all of them,
      // reduce this lane's row / column maxima from the landed raw stages, publish the
      // tables, then transform every stage in place (re-read from shared memory)
      int64_t g = 0;
      int lt = 0;
      for (int64_t t = blockIdx.x; t < grid.tiles; t += gridDim.x, ++lt, g += nk) {
        float ma0 = kNegInf, ma1 = kNegInf, mb = kNegInf;
        bool odd = false;
        for (int kb = 0; kb < nk; ++kb) {
          const int s = (int)((g + kb) % STAGES);
          mbar_wait(smem_u32(&full[s]), (uint32_t)(((g + kb) / STAGES) & 1));
          RawStage<G::kGroupsB> cur;
          load_stage<G::kGroupsB>(ring + s * G::kStage, xw, lane, cur);
          ma0 = fmaxf(ma0, fmaxf(cur.a0.x, cur.a0.z));
          ma1 = fmaxf(ma1, fmaxf(cur.a1.x, cur.a1.z));
          odd |= odd_phase(cur.a0.y) | odd_phase(cur.a0.w) | odd_phase(cur.a1.y) |
                 odd_phase(cur.a1.w);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            mb = fmaxf(mb, cur.b[0][j].x);
            odd |= odd_phase(cur.b[0][j].y);
          }
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
          ma0 = fmaxf(ma0, __shfl_xor_sync(0xffffffffu, ma0, o));
          ma1 = fmaxf(ma1, __shfl_xor_sync(0xffffffffu, ma1, o));
        }
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 8));
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 16));
        sa0 = fmaxf(ma0, 0.0f);
        sa1 = fmaxf(ma1, 0.0f);
        sb[0] = fmaxf(mb, 0.0f);
        const bool canon = !__any_sync(0xffffffffu, odd);
        const int slot = lt & (kScaleSlots - 1);
        if (bn == 0) {
          rowS[slot * BM + xw * 8 + r] = sa0;
          rowS[slot * BM + xw * 8 + r + 4] = sa1;
        }
        if (lane < 8) colS[slot * BN + xw * 8 + bn] = sb[0];
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&sc_full[slot]));
        for (int kb = 0; kb < nk; ++kb) {
          const int s = (int)((g + kb) % STAGES);
          RawStage<G::kGroupsB> cur;
          load_stage<G::kGroupsB>(ring + s * G::kStage, xw, lane, cur);
          if (canon)
            store_stage<G::kGroupsB, true>(ring + s * G::kStage, xw, lane, cur, sa0, sa1, sb);
          else
            store_stage<G::kGroupsB, false>(ring + s * G::kStage, xw, lane, cur, sa0, sa1, sb);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&ready[s]));
        }
      }
    } else if constexpr (kFuse) {
      // scale stages: running maxima of this lane's A rows (r, r + 4 of group xw) and B
      // column (bn of group xw) over its k; at a tile's last K-block, reduce over the lanes
      // sharing them, clamp at 0 and publish (core.py:252-253)
      float ma0 = kNegInf, ma1 = kNegInf, mb = kNegInf;
      bool odd = false, canon = false;
      int64_t lt_scale = 0;  // local index of the tile the scale stages belong to
      RingBits<STAGES> rb;
      int gpos = 0;
      FuseSeq q(blockIdx.x, gridDim.x, grid.tiles, nk, late);
      // no cross-stage software pipeline here: a main stage must not wait for the scale
      // stage behind it (an HBM read) before it is transformed; the 16 warps hide LDS latency
      for (; q.valid(); q.next()) {
        const int s = rb.s;
        const bool sc = q.scale();
        RawStage<G::kGroupsB> cur;
        if (xw == 0 && lane == 0) TC_TRACE(1, gpos, clock64());
        mbar_wait(smem_u32(&full[s]), rb.bit(rb.full));
        if (xw == 0 && lane == 0) TC_TRACE(2, gpos, clock64());
        if (sc && rowsA)
          load_stage_b<G::kGroupsB>(ring + s * G::kStage, xw, lane, cur);
        else
          load_stage<G::kGroupsB>(ring + s * G::kStage, xw, lane, cur);
        if (sc) {
          if (rowsA) {
            // this warp's rows 8 xw .. 8 xw + 7 as float4 indices [lo, hi) of the tile, the
            // part of them in chunk kb; one warp instruction never straddles a row (k % 64)
            const int k2 = k >> 1, c0 = q.block() * (G::kBytesA / 16);
            const int lo = max(8 * xw * k2, c0), hi = min((8 * xw + 8) * k2, c0 + G::kBytesA / 16);
            const uint32_t base = ring + s * G::kStage;
            for (int f = lo; f < hi; f += 32) {
              const float4 v = ld_shared_v4(base + (uint32_t)(f - c0 + lane) * 16u);
              odd |= odd_phase(v.y) | odd_phase(v.w);
              const float w = warp_max(fmaxf(v.x, v.z));
              if (lane == f / k2 - 8 * xw) ma0 = fmaxf(ma0, w);  // lane i: row 8 xw + i
            }
          } else {
            ma0 = fmaxf(ma0, fmaxf(cur.a0.x, cur.a0.z));
            ma1 = fmaxf(ma1, fmaxf(cur.a1.x, cur.a1.z));
            odd |= odd_phase(cur.a0.y) | odd_phase(cur.a0.w) | odd_phase(cur.a1.y) |
                   odd_phase(cur.a1.w);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            mb = fmaxf(mb, cur.b[0][j].x);
            odd |= odd_phase(cur.b[0][j].y);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&sfreed[s]));
          if (q.block() == nk - 1) {
            if (rowsA) {  // rows r, r + 4 of the group from lanes r, r + 4
              const float m8 = ma0;
              ma0 = __shfl_sync(0xffffffffu, m8, r);
              ma1 = __shfl_sync(0xffffffffu, m8, r + 4);
            } else {
#pragma unroll
              for (int o = 1; o < 8; o <<= 1) {
                ma0 = fmaxf(ma0, __shfl_xor_sync(0xffffffffu, ma0, o));
                ma1 = fmaxf(ma1, __shfl_xor_sync(0xffffffffu, ma1, o));
              }
            }
            mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 8));
            mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 16));
            sa0 = fmaxf(ma0, 0.0f);
            sa1 = fmaxf(ma1, 0.0f);
            sb[0] = fmaxf(mb, 0.0f);
            canon = !__any_sync(0xffffffffu, odd);
            const int slot = (int)(lt_scale & (kScaleSlots - 1));
            if (bn == 0) {
              rowS[slot * BM + xw * 8 + r] = sa0;
              rowS[slot * BM + xw * 8 + r + 4] = sa1;
            }
            if (lane < 8) colS[slot * BN + xw * 8 + bn] = sb[0];
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&sc_full[slot]));  // release.cta: tables
            ma0 = ma1 = mb = kNegInf;
            odd = false;
            ++lt_scale;
          }
        } else {
          if (canon)
            store_stage<G::kGroupsB, true>(ring + s * G::kStage, xw, lane, cur, sa0, sa1, sb);
          else
            store_stage<G::kGroupsB, false>(ring + s * G::kStage, xw, lane, cur, sa0, sa1, sb);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&ready[s]));
        }
        if (xw == 0 && lane == 0) TC_TRACE(4, gpos, clock64());
        rb.advance(sc);
        ++gpos;
      }
    } else {
      const bool canon = noncanon != nullptr && *noncanon == 0;
      int64_t t = blockIdx.x;
      auto load_scales = [&](int64_t tile) {
        int64_t b;
        int row0, col0;
        grid.at(tile, b, row0, col0, BN);
        const float* ra = rowA.at(b) + row0;
        const float* cb = colB.at(b) + col0;
        sa0 = ra[xw * 8 + r];
        sa1 = ra[xw * 8 + r + 4];
        sb[0] = cb[xw * 8 + bn];
        sb[1] = (BN / 8 > kXformWarps) ? cb[(xw + kXformWarps) * 8 + bn] : 0.0f;
      };
      if (t < grid.tiles) {
        load_scales(t);
        RawStage<G::kGroupsB> cur, nxt;
        mbar_wait(smem_u32(&full[0]), 0);
        load_stage<G::kGroupsB>(ring, xw, lane, cur);
        int kb = 0;
        for (int64_t g = 0;; ++g) {
          // position of stage g+1 (may belong to this CTA's next tile)
          int64_t tn = t;
          int kbn = kb + 1;
          if (kbn == nk) {
            kbn = 0;
            tn += gridDim.x;
          }
          const bool more = tn < grid.tiles;
          const int s = (int)(g % STAGES);
          if (more) {
            const int sn = (int)((g + 1) % STAGES);
            mbar_wait(smem_u32(&full[sn]), (uint32_t)(((g + 1) / STAGES) & 1));
            load_stage<G::kGroupsB>(ring + sn * G::kStage, xw, lane, nxt);
          }
          if (debug != 1 && debug != 3 && debug < 5) {
            if (canon)
              store_stage<G::kGroupsB, true>(ring + s * G::kStage, xw, lane, cur, sa0, sa1, sb);
            else
              store_stage<G::kGroupsB, false>(ring + s * G::kStage, xw, lane, cur, sa0, sa1, sb);
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&ready[s]));
          if (!more) break;
          if (tn != t) load_scales(tn);
          t = tn;
          kb = kbn;
          cur = nxt;
        }
      }
    }
  } else {
    // ------------------------------ epilogue ------------------------------
    const int e = warp - 2 - kXformWarps;
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = quad * 32 + lane;
    // this warp's accumulator columns (kDuo: the diagonal block of its rows' product only)
    const int half = quad >> 1;
    const int c_begin = kDuo ? 64 * half + 32 * (e >> 2) : (e >> 2) * G::kEpiCols;
    constexpr int kCols = kDuo ? 32 : G::kEpiCols;
    const uint32_t stage = ring + G::kOut + (uint32_t)(e * G::kStageOut);
    int lt = 0;
    for (int64_t t = blockIdx.x; t < grid.tiles; t += gridDim.x, ++lt) {
      int64_t b;
      int row0, col0;
      if constexpr (kDuo) {
        b = 2 * t + half;  // this warp's product; its rows / columns start at 64 * half
        row0 = col0 = -64 * half;
      } else {
        grid.at(t, b, row0, col0, BN);
      }
      const bool live = !kDuo || b < grid.batch;
      const int buf = lt & 1;
      if (e == 0 && lane == 0) TC_TRACE(5, lt, clock64());
      mbar_wait(smem_u32(&acc_full[buf]), (uint32_t)((lt >> 1) & 1));
      tc_fence_after();
      if (e == 0 && lane == 0) TC_TRACE(6, lt, clock64());
      float ai;
      const float* cb;
      if constexpr (kFuse) {
        const int slot = lt & (kScaleSlots - 1);
        mbar_wait(smem_u32(&sc_full[slot]), (uint32_t)((lt >> 2) & 1));
        ai = rowS[slot * BM + row];
        cb = colS + slot * BN;
      } else {
        ai = rowA.at(b)[row0 + row];
        cb = colB.at(b) + col0;
      }
      float2* cblk = C + b * strideC + (int64_t)(row0 + quad * 32) * m + col0;
      const float2* drow = D.ptr ? D.at(b) + (int64_t)(row0 + row) * m + col0 : nullptr;
      uint32_t rmax = 0;  // bits of max(log, 0): non-negative floats order like uints
#pragma unroll 1
      for (int col = c_begin; col < (debug == 7 || !live ? c_begin : c_begin + kCols); col += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * BN + col), v);
        // kSub columns per staging round: [32 rows][kSub] complex64, 16-byte chunks XOR-swizzled
        // by the row (conflict-free both ways)
        constexpr int kSub = G::kStageOut / 256;
        constexpr int kChunks = kSub / 2;  // 16-byte chunks per staged row
#pragma unroll
        for (int h = 0; h < 32; h += kSub) {
#pragma unroll
          for (int j = h; j < h + kSub; j += 2) {
            float2 o0 = tc_out(__uint_as_float(v[j]), ai, cb[col + j]);
            float2 o1 = tc_out(__uint_as_float(v[j + 1]), ai, cb[col + j + 1]);
            if (drow) {
              o0 = gadd_elem(o0, drow[col + j]);
              o1 = gadd_elem(o1, drow[col + j + 1]);
            }
            // (no memory clobber: the column-scale loads above may be hoisted past it)
            // TMA path: SWIZZLE_64B (chunk c of row r at c ^ ((r >> 1) & 3)), else c ^ r
            const int cs = G::kTmaOut ? (((j - h) >> 1) ^ (lane >> 1)) & 3
                                      : (((j - h) >> 1) ^ lane) & (kChunks - 1);
            st_shared_v4_staging(stage + lane * (kSub * 8) + (cs << 4),
                                 __float_as_uint(o0.x), __float_as_uint(o0.y),
                                 __float_as_uint(o1.x), __float_as_uint(o1.y));
            const uint32_t c0 = __float_as_uint(fmaxf(o0.x, 0.0f));
            const uint32_t c1 = __float_as_uint(fmaxf(o1.x, 0.0f));
            rmax = max(rmax, max(c0, c1));
            if (emit.col) {
              const uint32_t m0 = __reduce_max_sync(0xffffffffu, c0);
              const uint32_t m1 = __reduce_max_sync(0xffffffffu, c1);
              if (lane == 0) {
                unsigned int* cc = reinterpret_cast<unsigned int*>(emit.col + b * emit.col_stride +
                                                                   col0 + col + j);
                atomicMax(cc, m0);
                atomicMax(cc + 1, m1);
              }
            }
          }
          if constexpr (G::kTmaOut) {
            // the staging buffer is the 128B-swizzled box of mapC: one TMA store per 32 x 16
            fence_async_smem();
            __syncwarp();
            if (lane == 0 && debug != 8) {
              if (hints)  // the output streams out: evict_first
                tma_store_3d_hint(&mapC, stage, col0 + col + h, row0 + quad * 32, (int)b, pol_drop);
              else
                tma_store_3d(&mapC, stage, col0 + col + h, row0 + quad * 32, (int)b);
              tma_store_wait_read<0>();  // the buffer is rewritten by the next sub-chunk
            }
            __syncwarp();
          } else {
            __syncwarp();
            // copy-out: full kSub * 8-byte row segments, 512 B per instruction (coalesced),
            // where a lane-per-row store would touch 32 lines per instruction
            constexpr int kRowsPer = 32 / kChunks;  // rows per instruction
#pragma unroll 4
            for (int it = 0; it < 32 / kRowsPer; ++it) {
              const int rr = kRowsPer * it + lane / kChunks, c = lane & (kChunks - 1);
              const float4 o =
                  ld_shared_v4(stage + rr * (kSub * 8) + (((c ^ rr) & (kChunks - 1)) << 4));
              if (debug != 8) *reinterpret_cast<float4*>(cblk + (int64_t)rr * m + col + h + 2 * c) = o;
            }
            __syncwarp();
          }
        }
      }
      if (!kDuo && emit.row)
        atomicMax(reinterpret_cast<unsigned int*>(emit.row + b * emit.row_stride + row0 + row), rmax);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&acc_empty[buf]));
      if (e == 0 && lane == 0) TC_TRACE(7, lt, clock64());
    }
    if (G::kTmaOut && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(G::kTmemCols));
  }
}

// GOOM_TC_DEBUG (profiling only; results invalid): 1 skips the transform, 2 the MMAs,
// 3 the TMA loads and the transform, 4 the TMA loads, 5 transform and MMAs (TMA ring only),
// 6 as 5 with B loaded as full-width rows, 7 skips the epilogue, 8 its global stores
// (the kFuse kernel honours 6, 7 and 8 only)
int tc_debug() {
  static int v = [] {
    const char* e = getenv("GOOM_TC_DEBUG");
    const char* p = getenv("GOOM_TC_PREFETCH");  // kFuse: L2 prefetch distance in tiles
    return (e ? atoi(e) : 0) | (((p ? atoi(p) : 0) & 15) << 8) |
           ((fuse_lateness("GOOM_TC1_LATE", 1) & 15) << 12);  // (fitted per launch)
  }();
  return v;
}

template <int BN, bool kFuse, bool kDuo = false>
int launch_tc(const LmmeProblem& p, cudaStream_t s) {
  using G = Cfg<BN, kFuse>;
  GOOM_TRY(smem_attr((const void*)lmme_tc_kernel<BN, kFuse, kDuo>, G::kSmem, "lmme_tc smem attribute"));
  constexpr int kRowsBox = kDuo ? BM / 2 : BM;  // kDuo: each product half is its own box
  alignas(64) CUtensorMap mapA, mapB;
  int64_t mats, mstride;
  // A: (k, n, matrix) complex64 moved as int64, box 16 k x 128 rows
  mats_of(p.A, p.batch, p.n, p.k, mats, mstride);
  {
    cuuint64_t dims[3] = {(cuuint64_t)p.k, (cuuint64_t)p.n, (cuuint64_t)mats};
    cuuint64_t strides[2] = {(cuuint64_t)p.k * 8, (cuuint64_t)mstride * 8};
    cuuint32_t box[3] = {BK, kRowsBox, 1};
    GOOM_TRY(encode(&mapA, p.A, 3, dims, strides, box));
  }
  // B: (8 cols, k, m/8 column groups, matrix), box 8 x 16 k x BN/8 -> [group][k][8] in smem
  mats_of(p.B, p.batch, p.k, p.m, mats, mstride);
  {
    cuuint64_t dims[4] = {8, (cuuint64_t)p.k, (cuuint64_t)(p.m / 8), (cuuint64_t)mats};
    cuuint64_t strides[3] = {(cuuint64_t)p.m * 8, 64, (cuuint64_t)mstride * 8};
    cuuint32_t box[4] = {8, BK, (kDuo ? BN / 2 : BN) / 8, 1};
    GOOM_TRY(encode(&mapB, p.B, 4, dims, strides, box));
  }
  alignas(64) CUtensorMap mapB3;  // GOOM_TC_DEBUG=6 only: B as [16 k][BN] rows of BN*8 bytes
  {
    cuuint64_t dims[3] = {(cuuint64_t)p.m, (cuuint64_t)p.k, (cuuint64_t)mats};
    cuuint64_t strides[2] = {(cuuint64_t)p.m * 8, (cuuint64_t)mstride * 8};
    cuuint32_t box[3] = {BN, BK, 1};
    GOOM_TRY(encode(&mapB3, p.B, 3, dims, strides, box));
  }
  // C: (m, n, batch) complex64 as int64, box 8 cols x 32 rows, 64B swizzle (TMA epilogue)
  alignas(64) CUtensorMap mapC;
  if (G::kTmaOut) {
    if ((reinterpret_cast<uintptr_t>(p.C) & 15) || (p.strideC & 1))
      return fail(GOOM_EUNSUPPORTED, "lmme_tc: output not 16-byte aligned");
    const int64_t cb = p.strideC == 0 ? 1 : p.batch;
    const int64_t cs = p.strideC == 0 ? (int64_t)p.n * p.m : p.strideC;
    cuuint64_t dims[3] = {(cuuint64_t)p.m, (cuuint64_t)p.n, (cuuint64_t)cb};
    cuuint64_t strides[2] = {(cuuint64_t)p.m * 8, (cuuint64_t)cs * 8};
    cuuint32_t box[3] = {8, 32, 1};
    GOOM_TRY(encode(&mapC, Operand{p.C, 0, 1}, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B));
  }
  TileGrid tg;
  tg.nct = kDuo ? 1 : p.m / BN;
  tg.nrt = kDuo ? 1 : p.n / BM;
  tg.b_base = 0;
  tg.batch = p.batch;
  tg.tiles = kDuo ? (p.batch + 1) / 2 : p.batch * tg.nct * tg.nrt;
  const int64_t sms = num_sms();
  const unsigned grid = (unsigned)(tg.tiles < sms ? tg.tiles : sms);
  Emit emit{p.emitRow, p.emitRowStride, p.emitCol, p.emitColStride};
  lmme_tc_kernel<BN, kFuse, kDuo><<<grid, G::kThreads, G::kSmem, s>>>(
      mapA, mapB, mapB3, mapC, p.A, p.B, p.D, p.rowA, p.colB, p.C, p.strideC, tg, p.n, p.k, p.m, p.noncanon,
      emit, (tc_debug() & ~(15 << 12)) | (fit_lateness((tc_debug() >> 12) & 15, p.k / BK) << 12));
  GOOM_CHECK_LAUNCH("lmme_tc_kernel");
  return GOOM_OK;
}

// GOOM_TC_FUSE: 1 always reduce the scales in the one-SM kernel when the caller gives none,
// 0 never (pre-pass); unset: when a product is a single 128 x 128 tile (n == m == 128: the
// HBM-bound config-2 shape), so the scale pass reads nothing a second time from HBM
int tc_fuse_mode() {
  static int v = [] {
    const char* e = getenv("GOOM_TC_FUSE");
    return e ? atoi(e) : -1;
  }();
  return v;
}

}  // namespace

bool lmme_tc_eligible(int n, int k, int m) {
  return n > 0 && k > 0 && m > 0 && n % BM == 0 && m % 128 == 0 && k % BK == 0;
}

// the one-SM kernel's scale pass: BN = 128 tiles, >= 4 K-blocks (the 4-slot scale tables are
// recycled only after the MMA of a later tile has started, which 4 K-blocks guarantee)
bool lmme_tc1_fuse_scales(int n, int k, int m) {
  if (!lmme_tc_eligible(n, k, m) || k < 4 * BK) return false;
  const int f = tc_fuse_mode();
  return f == 1 || (f < 0 && n == 128 && m == 128);
}

// n = m = 64 (config 2's smallest shape): two products per 128 x 128 tile, A rows
// [product 2t | product 2t + 1], B columns likewise; the MMA also forms the two cross blocks,
// which the epilogue drops (the tensor core has the headroom: the shape is HBM-bound).
// k = 64: a tile's four K-blocks (128 KB) fit the ring, so they are loaded ONCE and the
// transform reduces the clamped scales from the landed stages before transforming them
// (no second read). No row / column emission.
bool lmme_tc_duo_eligible(int n, int k, int m) {
  return n == 64 && m == 64 && k == 64 && tc_fuse_mode() != 0;  // a tile's K-blocks fit the ring
}

int lmme_tc_duo(const LmmeProblem& p, cudaStream_t s) {
  if (!lmme_tc_duo_eligible(p.n, p.k, p.m) || p.rowA.ptr || p.colB.ptr || p.emitRow || p.emitCol)
    return GOOM_EUNSUPPORTED;
  if (((reinterpret_cast<uintptr_t>(p.A.ptr) | reinterpret_cast<uintptr_t>(p.B.ptr)) & 15) ||
      ((p.A.stride | p.B.stride) & 1))
    return GOOM_EUNSUPPORTED;
  return launch_tc<128, true, true>(p, s);
}

int lmme_tc(const LmmeProblem& p, cudaStream_t s) {
  if (!lmme_tc_eligible(p.n, p.k, p.m)) return GOOM_EUNSUPPORTED;
  // TMA: 16-byte aligned bases and matrix strides
  if (((reinterpret_cast<uintptr_t>(p.A.ptr) | reinterpret_cast<uintptr_t>(p.B.ptr)) & 15) ||
      ((p.A.stride | p.B.stride) & 1))
    return GOOM_EUNSUPPORTED;
  static const bool pairs = [] {
    const char* e = getenv("GOOM_TC2");
    return !(e && atoi(e) == 0);
  }();
  if (pairs && lmme_tc2_eligible(p.n, p.k, p.m)) {
    const int rc = lmme_tc2(p, s);
    if (rc != GOOM_EUNSUPPORTED) return rc;
  }
  if (!p.rowA.ptr || !p.colB.ptr) {
    if (!lmme_tc1_fuse_scales(p.n, p.k, p.m)) return GOOM_EUNSUPPORTED;
    return launch_tc<128, true>(p, s);
  }
  if (p.m % 256 == 0) return launch_tc<256, false>(p, s);
  return launch_tc<128, false>(p, s);
}

}  // namespace goom

#ifdef GOOM_TC_TRACE
extern "C" int goom_tc_trace_read(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, goom::g_tc_trace, sizeof(goom::g_tc_trace));
}
#endif
