// tcgen05 LMME on CTA pairs (cta_group::2): the complex64 LMME of Eq. 10-12 with the
// real GEMM at FP32 accuracy (3xTF32) for n, m multiples of 256 — the shape of every
// combine in the d = 512 / 1024 chain scans.
//
// Why pairs (measured on B200, profiles/r1_ubench_tcgen05_tf32_smem.txt): a kind::tf32
// 128x256x8 MMA takes 128 clk and, at cta_group::1, reads 96 B/clk of shared memory
// through the same read port as LDS; the in-kernel GOOM -> TF32 transform must LDS the
// raw complex64 K-block (another ~62 B/clk at full MMA rate), so the one-SM kernel
// (lmme_tc.cu) cannot exceed ~80% of the tensor rate even with perfect overlap. A
// 256x256 pair tile halves the per-SM B panel: the MMA reads 64 B/clk per SM and the
// transform 42 B/clk, under the 128 B/clk port; the per-SM transform work per MAC also
// drops by 1/3 (128 + 128 operand rows per 128 x 256 accumulator instead of 128 + 256).
//
// Pair tile = 256 rows x 256 columns, full K. CTA r (= %cluster_ctarank) owns rows
// 128r..128r+127 of the A panel, columns 128r..128r+127 of the B panel, and rows
// 128r.. of the accumulator (all 256 columns, in its own TMEM). Per CTA:
//   warp 0        TMA loader: raw complex64 K-block (16 k) of its A half (16 groups of
//                 [8 rows][16 k]) and of its B half (16 groups of [16 k][8 cols], rows
//                 landed in k-order (4*(s%4) + s/4) so the transform's column gathers
//                 are bank-conflict-free);
//   warp 1        (leader CTA) MMA issuer: 6 x tcgen05.mma.cta_group::2.kind::tf32
//                 (M=256, N=256, K=8) per K-block: small*big + big*small + big*big;
//   warps 2..17   transform, in place: v = sign * exp(log - scale) -> (big, small) TF32
//                 planes in the 64B-swizzled K-major layout; arrive on the LEADER's
//                 ready barrier (remote arrive from CTA 1);
//   warps 18..21  epilogue: tcgen05.ld of this CTA's 128 accumulator rows,
//                 (log|I| + a_i) + b_j and the sign, optional fused gadd, store, and the
//                 clamped row / column maxima of C for the next LMME (atomicMax).
// Stages are released by tcgen05.commit multicast to both CTAs; the accumulator is
// double-buffered (2 x 256 TMEM columns) so the epilogue of tile i overlaps tile i+1.
// Persistent: grid = 2 x (co-resident clusters), pair tiles strided over clusters.
#include <cstdlib>

#include "tc_ptx.cuh"

namespace goom {

namespace {
using namespace tc;

constexpr int kRowsCta = 128;            // accumulator rows per CTA (M = 256 per pair)
constexpr int kPairN = 256;              // N per pair tile (128 B columns per CTA)
constexpr int BK = 16;
constexpr int kXformWarps = 16;
constexpr int kEpiWarps = 4;
constexpr int kThreads = 64 + (kXformWarps + kEpiWarps) * 32;  // 704
constexpr int kBytesA = (kRowsCta / 8) * kGroupBytes;          // 16 KB
constexpr int kBytesB = (kPairN / 2 / 8) * kGroupBytes;         // 16 KB
constexpr int kStage = kBytesA + kBytesB;                       // 32 KB
constexpr int kTmemCols = 2 * kPairN;                           // 512: double buffer
constexpr int kStageOut = 32 * 16 * 8;                         // 4 KB: 32 rows x 16 cols c64
constexpr int kOutBytes = kEpiWarps * 2 * kStageOut;            // 32 KB: 2 buffers per warp
// kFuse (scales reduced in-kernel, no pre-pass): every K-block is loaded twice through the
// ring, once a tile ahead as a SCALE stage (the transform warps reduce the maxima of exactly
// the A rows / B columns they later transform) and once for the main loop (lmme_tc.cu kFuse,
// FuseSeq); a 4-slot ring of per-tile tables (this CTA's 128 row scales, the pair tile's 256
// column scales, the peer's half written over DSMEM) feeds the epilogue
constexpr int kScaleSlots = 4;
constexpr int kScaleBytes = kScaleSlots * (kRowsCta + kPairN) * 4;
template <bool kFuse>
struct Tc2Cfg {
  static constexpr int S = kFuse ? 5 : 6;                       // ring stages
  static constexpr int kRing = S * kStage;                      // 160 / 192 KB
  static constexpr int kScaleOff = kRing + kOutBytes;
  static constexpr int kBarOff = kScaleOff + (kFuse ? kScaleBytes : 0);
  static constexpr int kSmem = kBarOff + 1024 /*align*/ + 512 /*barriers*/;
};

// (cluster / pair helpers: tc_ptx.cuh)

// Raw K-block slice of one transform warp: A group xw (lane: rows l/8 and 4 + l/8, k-pair
// l%8) and B group xw (lane (n = l%8, c = l/8): k = 4c..4c+3 of column n, landed at smem
// rows c + 4j so each LDS.64 covers 4 consecutive 64-byte rows: conflict-free).
// ring position (stage, phase parity) advanced incrementally: no divisions in the loops
template <int kStages>
struct RingPos {
  int s = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next() {
    if (++s == kStages) {
      s = 0;
      ph ^= 1u;
    }
  }
};

struct Raw {
  float4 a0, a1;
  float2 b[4];
};

__device__ __forceinline__ void load_raw(uint32_t stage, int xw, int lane, Raw& r) {
  const uint32_t ga = stage + xw * kGroupBytes;
  r.a0 = ld_shared_v4(ga + lane * 16);
  r.a1 = ld_shared_v4(ga + 512 + lane * 16);
  const uint32_t gb = stage + kBytesA + xw * kGroupBytes;
  const int bn = lane & 7, bc = lane >> 3;
#pragma unroll
  for (int j = 0; j < 4; ++j) r.b[j] = ld_shared_v2(gb + (bc + 4 * j) * 64 + bn * 8);
}

template <bool kCanon>
__device__ __forceinline__ void store_planes(uint32_t stage, int xw, int lane, const Raw& r,
                                             float sa0, float sa1, float sb) {
  uint32_t ha[4], la[4], hb[4], lb[4];
  goom_split<kCanon>(make_float2(r.a0.x, r.a0.y), sa0, ha[0], la[0]);
  goom_split<kCanon>(make_float2(r.a0.z, r.a0.w), sa0, ha[1], la[1]);
  goom_split<kCanon>(make_float2(r.a1.x, r.a1.y), sa1, ha[2], la[2]);
  goom_split<kCanon>(make_float2(r.a1.z, r.a1.w), sa1, ha[3], la[3]);
#pragma unroll
  for (int j = 0; j < 4; ++j) goom_split<kCanon>(r.b[j], sb, hb[j], lb[j]);
  __syncwarp();  // the whole group is in registers before any of it is overwritten
  const int rr = lane >> 3, kp = lane & 7;
  const uint32_t ga = stage + xw * kGroupBytes;
  const uint32_t o0 = sw64_off(rr, kp >> 1) + (kp & 1) * 8;
  const uint32_t o1 = sw64_off(rr + 4, kp >> 1) + (kp & 1) * 8;
  st_shared_v2(ga + o0, ha[0], ha[1]);
  st_shared_v2(ga + 512 + o0, la[0], la[1]);
  st_shared_v2(ga + o1, ha[2], ha[3]);
  st_shared_v2(ga + 512 + o1, la[2], la[3]);
  const uint32_t gb = stage + kBytesA + xw * kGroupBytes;
  const uint32_t ob = sw64_off(lane & 7, lane >> 3);
  st_shared_v4(gb + ob, hb[0], hb[1], hb[2], hb[3]);
  st_shared_v4(gb + 512 + ob, lb[0], lb[1], lb[2], lb[3]);
}

// DSMEM store into CTA `rank` of the cluster at this CTA's shared offset
__device__ __forceinline__ void st_cluster_f32(uint32_t local, uint32_t rank, float v) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank));
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(remote), "f"(v) : "memory");
}
// release at cluster scope: the DSMEM stores before it are visible to the waiter
__device__ __forceinline__ void mbar_arrive_release_cluster(uint32_t bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_acquire_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, 0x989680;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

struct PairGrid {
  int nct, nrt;    // pair-tile columns / rows per product
  int64_t tiles;   // pair tiles in this launch
  __device__ __forceinline__ void at(int64_t t, int64_t& b, int& prow0, int& pcol0) const {
    const int ct = (int)(t % nct);
    const int64_t q = t / nct;
    prow0 = (int)(q % nrt) * 256;
    pcol0 = ct * kPairN;
    b = q / nrt;
  }
};

struct Emit {
  float* row;
  int64_t row_stride;
  float* col;
  int64_t col_stride;
};

template <bool kFuse>
__global__ void __launch_bounds__(kThreads, 1)
    lmme_tc2_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    const __grid_constant__ CUtensorMap mapC,
                    Operand A, Operand B, Operand D, Scales rowA, Scales colB,
                    float2* __restrict__ C, int64_t strideC, PairGrid grid, int k, int m,
                    const int* __restrict__ noncanon, Emit emit, int debug) {
  using Cfg = Tc2Cfg<kFuse>;
  constexpr int kStages = Cfg::S, kRing = Cfg::kRing;
  using Ring = RingPos<kStages>;
  // kFuse: a late scale pass (FuseSeq lateness, GOOM_TC_LATE, default 8 per main stage in the
  // tile's last 1/8) — scale-read lines wait less than a tile in L2 for their main-pass re-read
  // (d = 256: one per main stage 422 us, DRAM reads 2.02 GB; lateness 2 397 us, 1.50 GB;
  // lateness 8 390 us); GOOM_TC_DEBUG bit 64 restores one per main stage
  const int late = (debug & 64) ? 1 : ((debug >> 8) & 15);  // FuseSeq lateness (GOOM_TC_LATE)
  debug &= 63;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kBarOff);
  uint64_t* full = bars;                    // [S] local: TMA bytes landed
  uint64_t* ready = bars + kStages;         // [S] leader: both CTAs' stage transformed
  uint64_t* freed = bars + 2 * kStages;     // [S] local: stage's MMAs retired (multicast)
  uint64_t* acc_full = bars + 3 * kStages;  // [2] local: accumulator complete (multicast)
  uint64_t* acc_empty = acc_full + 2;       // [2] leader: both CTAs drained the buffer
  uint64_t* sc_full = acc_empty + 2;        // [4] kFuse: a tile's scale tables complete
  uint64_t* sfreed = sc_full + kScaleSlots;  // [S] kFuse local: scale stage read (16 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sfreed + kStages);
  // kFuse scale area: rowS [slot][128], colS [slot][256], column-max scratch, flags
  float* rowS = reinterpret_cast<float*>(smem + Cfg::kScaleOff);
  float* colS = rowS + kScaleSlots * kRowsCta;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cta_rank();
  const int64_t cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int nk = k / BK;

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
    if (kFuse) {  // every transform warp of both CTAs publishes its part of a tile's tables
      for (int i = 0; i < kScaleSlots; ++i) mbar_init(smem_u32(&sc_full[i]), 2 * kXformWarps);
      for (int i = 0; i < kStages; ++i) mbar_init(smem_u32(&sfreed[i]), kXformWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // one warp of EACH CTA takes part in the pair allocation
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // barriers of both CTAs initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t ring = smem_u32(smem);

  if (warp == 0) {
    // ------------------------------ loader (both CTAs) ------------------------------
    if (kFuse && lane == 0) {
      // scale pass one tile ahead through the same ring (lmme_tc.cu kFuse, FuseSeq): scale
      // stages keep their lines in L2 for the main pass, which frees them
      const uint64_t pol_keep = policy_evict_last(), pol_drop = policy_evict_first();
      RingBits<kStages> rb;
      int64_t ct = -1;
      int row0 = 0, col0 = 0, ma = 0, mb = 0;
      int64_t ct2 = -1;
      int row02 = 0, col02 = 0, ma2 = 0, mb2 = 0;
      for (FuseSeq q(cluster, nclusters, grid.tiles, nk, late); q.valid(); q.next()) {
        const int s = rb.s;
        if (rb.bit(rb.used)) {
          if (rb.bit(rb.last_scale))
            mbar_wait(smem_u32(&sfreed[s]), rb.bit(rb.scalep) ^ 1u);
          else
            mbar_wait(smem_u32(&freed[s]), rb.bit(rb.mainp) ^ 1u);
        }
        const bool sc = q.scale();
        // coordinates once per tile (one thread: no int64 divisions per stage)
        int64_t& tt = sc ? ct2 : ct;
        int &r0 = sc ? row02 : row0, &c0 = sc ? col02 : col0, &a0 = sc ? ma2 : ma,
            &b0 = sc ? mb2 : mb;
        if (tt != q.tile()) {
          tt = q.tile();
          int64_t b;
          int prow0, pcol0;
          grid.at(tt, b, prow0, pcol0);
          r0 = prow0 + (int)rank * kRowsCta;
          c0 = pcol0 + (int)rank * (kPairN / 2);
          a0 = A.stride == 0 ? 0 : (int)(b / A.div);
          b0 = B.stride == 0 ? 0 : (int)(b / B.div);
        }
        const uint32_t bar = smem_u32(&full[s]);
        mbar_expect_tx(bar, kStage);
        const uint32_t dst = ring + s * kStage;
        const int k0 = q.block() * BK;
        const uint64_t pol = sc ? pol_keep : pol_drop;
        tma_load_3d_hint(dst, &mapA, k0, r0, a0, bar, pol);
        tma_load_5d_hint(dst + kBytesA, &mapB, 0, k0 / 4, 0, c0 / 8, b0, bar, pol);
        rb.advance(sc);
      }
    } else if (lane == 0) {
      Ring rp;
      for (int64_t t = cluster; t < grid.tiles; t += nclusters) {
        int64_t b;
        int prow0, pcol0;
        grid.at(t, b, prow0, pcol0);
        const int row0 = prow0 + (int)rank * kRowsCta;
        const int col0 = pcol0 + (int)rank * (kPairN / 2);
        const int ma = A.stride == 0 ? 0 : (int)(b / A.div);
        const int mb = B.stride == 0 ? 0 : (int)(b / B.div);
        for (int kb = 0; kb < nk; ++kb, rp.next()) {
          const int s = rp.s;
          mbar_wait(smem_u32(&freed[s]), rp.ph ^ 1u);
          const uint32_t bar = smem_u32(&full[s]);
          if (debug >= 3 && debug != 5 && debug != 7) {  // profiling aid: no loads
            mbar_arrive(bar);
            continue;
          }
          mbar_expect_tx(bar, kStage);
          const uint32_t dst = ring + s * kStage;
          const int k0 = kb * BK;
          tma_load_3d(dst, &mapA, k0, row0, ma, bar);                              // [128][16 k]
          tma_load_5d(dst + kBytesA, &mapB, 0, k0 / 4, 0, col0 / 8, mb, bar);      // [16][4][4][8]
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------ MMA issuer (leader CTA) ------------------------------
    if (kFuse && rank == 0 && lane == 0) {
      constexpr uint32_t idesc = tf32_idesc(2 * kRowsCta, kPairN);
      RingBits<kStages> rb;
      int lt = -1;
      uint32_t acc = tmem;
      for (FuseSeq q(cluster, nclusters, grid.tiles, nk, late); q.valid(); q.next()) {
        const int s = rb.s;
        const bool sc = q.scale();
        if (!sc) {
          if (q.kb == 0) {
            ++lt;
            mbar_wait(smem_u32(&acc_empty[lt & 1]), (uint32_t)((lt >> 1) & 1) ^ 1u);
            tc_fence_after();
            acc = tmem + (uint32_t)((lt & 1) * kPairN);
          }
          mbar_wait(smem_u32(&ready[s]), rb.bit(rb.mainp));
          tc_fence_after();
          const uint32_t base = ring + s * kStage;
          const uint64_t dAb = sw64_desc(base), dAs = sw64_desc(base + 512);
          const uint64_t dBb = sw64_desc(base + kBytesA), dBs = sw64_desc(base + kBytesA + 512);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t adv = (uint64_t)(kk * 32) >> 4;
            mma_tf32_pair(acc, dAs + adv, dBb + adv, idesc, (q.kb | kk) != 0);
            mma_tf32_pair(acc, dAb + adv, dBs + adv, idesc, 1);
            mma_tf32_pair(acc, dAb + adv, dBb + adv, idesc, 1);
          }
          mma_commit_pair(smem_u32(&freed[s]));
          if (q.kb == nk - 1) mma_commit_pair(smem_u32(&acc_full[lt & 1]));
        }
        rb.advance(sc);
      }
    } else if (!kFuse && rank == 0 && lane == 0) {
      constexpr uint32_t idesc = tf32_idesc(2 * kRowsCta, kPairN);
      Ring rp;
      int lt = 0;
      for (int64_t t = cluster; t < grid.tiles; t += nclusters, ++lt) {
        const int buf = lt & 1;
        mbar_wait(smem_u32(&acc_empty[buf]), (uint32_t)((lt >> 1) & 1) ^ 1u);
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(buf * kPairN);
        for (int kb = 0; kb < nk; ++kb, rp.next()) {
          const int s = rp.s;
          mbar_wait(smem_u32(&ready[s]), rp.ph);
          tc_fence_after();
          if (debug != 2 && debug != 5 && debug != 7 && debug != 9) {
            const uint32_t base = ring + s * kStage;
            const uint64_t dAb = sw64_desc(base), dAs = sw64_desc(base + 512);
            const uint64_t dBb = sw64_desc(base + kBytesA), dBs = sw64_desc(base + kBytesA + 512);
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint64_t adv = (uint64_t)(kk * 32) >> 4;  // 8 TF32 = 32 B along K
              mma_tf32_pair(acc, dAs + adv, dBb + adv, idesc, (kb | kk) != 0);
              mma_tf32_pair(acc, dAb + adv, dBs + adv, idesc, 1);
              mma_tf32_pair(acc, dAb + adv, dBb + adv, idesc, 1);
            }
          }
          mma_commit_pair(smem_u32(&freed[s]));
        }
        mma_commit_pair(smem_u32(&acc_full[buf]));
      }
    }
    __syncwarp();
  } else if (warp < 2 + kXformWarps) {
    // ------------------------------ transform (both CTAs) ------------------------------
    const int xw = warp - 2;
    const int r8 = lane >> 3, bn = lane & 7;
    const uint32_t ready0 = smem_u32(&ready[0]);
    float sa0 = 0.f, sa1 = 0.f, sb = 0.f;
    if constexpr (kFuse) {
      // Eq. 11's clamped scales (core.py:252-253) from the scale stages: running maxima of
      // this lane's A rows (r8, r8 + 4 of group xw) and B column (bn of group xw); at the
      // tile's last K-block, reduced over the lanes sharing them, clamped at 0, published to
      // the epilogue tables (the column scales to both CTAs: each epilogue needs all 256)
      float ma0 = kNegInf, ma1 = kNegInf, mb = kNegInf;
      bool odd = false, canon = false;
      int lt_scale = 0;
      RingBits<kStages> rb;
      for (FuseSeq q(cluster, nclusters, grid.tiles, nk, late); q.valid(); q.next()) {
        const int s = rb.s;
        const bool sc = q.scale();
        Raw cur;
        mbar_wait(smem_u32(&full[s]), rb.bit(rb.full));
        load_raw(ring + s * kStage, xw, lane, cur);
        if (sc) {
          ma0 = fmaxf(ma0, fmaxf(cur.a0.x, cur.a0.z));
          ma1 = fmaxf(ma1, fmaxf(cur.a1.x, cur.a1.z));
          odd |= odd_phase(cur.a0.y) | odd_phase(cur.a0.w) | odd_phase(cur.a1.y) |
                 odd_phase(cur.a1.w);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            mb = fmaxf(mb, cur.b[j].x);
            odd |= odd_phase(cur.b[j].y);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&sfreed[s]));
          if (q.block() == nk - 1) {
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
              ma0 = fmaxf(ma0, __shfl_xor_sync(0xffffffffu, ma0, o));
              ma1 = fmaxf(ma1, __shfl_xor_sync(0xffffffffu, ma1, o));
            }
            mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 8));
            mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 16));
            sa0 = fmaxf(ma0, 0.0f);
            sa1 = fmaxf(ma1, 0.0f);
            sb = fmaxf(mb, 0.0f);
            canon = !__any_sync(0xffffffffu, odd);
            const int slot = lt_scale & (kScaleSlots - 1);
            if (bn == 0) {
              rowS[slot * kRowsCta + xw * 8 + r8] = sa0;
              rowS[slot * kRowsCta + xw * 8 + r8 + 4] = sa1;
            }
            if (lane < 8) {
              float* cs = colS + slot * kPairN + rank * (kPairN / 2) + xw * 8 + bn;
              *cs = sb;
              st_cluster_f32(smem_u32(cs), rank ^ 1u, sb);
            }
            __syncwarp();
            if (lane == 0) {
              mbar_arrive(smem_u32(&sc_full[slot]));                            // local tables
              mbar_arrive_release_cluster(smem_u32(&sc_full[slot]), rank ^ 1u);  // peer's
            }
            ma0 = ma1 = mb = kNegInf;
            odd = false;
            ++lt_scale;
          }
        } else {
          if (canon)
            store_planes<true>(ring + s * kStage, xw, lane, cur, sa0, sa1, sb);
          else
            store_planes<false>(ring + s * kStage, xw, lane, cur, sa0, sa1, sb);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive_rank(ready0 + s * 8, 0);
        }
        rb.advance(sc);
      }
    } else {
      const bool canon = noncanon != nullptr && *noncanon == 0;
      int64_t t = cluster;
      auto load_scales = [&](int64_t tile) {
        int64_t b;
        int prow0, pcol0;
        grid.at(tile, b, prow0, pcol0);
        const float* ra = rowA.at(b) + prow0 + rank * kRowsCta + xw * 8;
        sa0 = ra[r8];
        sa1 = ra[r8 + 4];
        sb = colB.at(b)[pcol0 + rank * (kPairN / 2) + xw * 8 + bn];
      };
      if (t < grid.tiles) {
        load_scales(t);
        Raw cur, nxt;
        mbar_wait(smem_u32(&full[0]), 0);
        load_raw(ring, xw, lane, cur);
        int kb = 0;
        Ring rc, rn;  // current stage and the next one
        rn.next();
        for (;;) {
          int64_t tn = t;
          int kbn = kb + 1;
          if (kbn == nk) {
            kbn = 0;
            tn += nclusters;
          }
          const bool more = tn < grid.tiles;
          const int s = rc.s;
          if (more) {
            mbar_wait(smem_u32(&full[rn.s]), rn.ph);
            load_raw(ring + rn.s * kStage, xw, lane, nxt);
          }
          if (debug == 0 || debug == 2 || debug == 4) {
            if (canon)
              store_planes<true>(ring + s * kStage, xw, lane, cur, sa0, sa1, sb);
            else
              store_planes<false>(ring + s * kStage, xw, lane, cur, sa0, sa1, sb);
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive_rank(ready0 + s * 8, 0);
          if (!more) break;
          rc.next();
          rn.next();
          if (tn != t) load_scales(tn);
          t = tn;
          kb = kbn;
          cur = nxt;
        }
      }
    }
  } else {
    // ------------------------------ epilogue (both CTAs) ------------------------------
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = quad * 32 + lane;
    const uint32_t obuf = smem_u32(smem + kRing) + (uint32_t)(warp - 2 - kXformWarps) * 2 * kStageOut;
    const uint32_t acc_empty0 = smem_u32(&acc_empty[0]);
    const uint64_t pol_out = policy_evict_first();
    int lt = 0;
    for (int64_t t = cluster; t < grid.tiles; t += nclusters, ++lt) {
      int64_t b;
      int prow0, pcol0;
      grid.at(t, b, prow0, pcol0);
      const int buf = lt & 1;
      mbar_wait(smem_u32(&acc_full[buf]), (uint32_t)((lt >> 1) & 1));
      tc_fence_after();
      const int grow = prow0 + (int)rank * kRowsCta + row;
      float ai;
      const float* cb;
      if constexpr (kFuse) {
        const int slot = lt & (kScaleSlots - 1);
        mbar_wait_acquire_cluster(smem_u32(&sc_full[slot]), (uint32_t)((lt >> 2) & 1));
        ai = rowS[slot * kRowsCta + row];
        cb = colS + slot * kPairN;
      } else {
        ai = rowA.at(b)[grow];
        cb = colB.at(b) + pcol0;
      }
      const float2* drow = D.ptr ? D.at(b) + (int64_t)grow * m + pcol0 : nullptr;
      uint32_t rmax = 0;  // bits of max(log, 0): non-negative floats order like uints
      const int wrow0 = prow0 + (int)rank * kRowsCta + quad * 32;  // this warp's 32 rows
#pragma unroll 1
      for (int col = 0; col < (debug == 7 || debug == 8 ? 0 : kPairN); col += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * kPairN + col), v);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          // staging buffer (col/16) & 1: the TMA store issued two sub-chunks ago has read it
          const uint32_t sbuf = obuf + (uint32_t)(((col >> 4) + h) & 1) * kStageOut;
          if (lane == 0) tma_store_wait_read<1>();
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            const int cc = col + 16 * h + j;
            const float4 s4 = *reinterpret_cast<const float4*>(cb + cc);  // uniform: broadcast
            float2 o0 = tc_out(__uint_as_float(v[16 * h + j]), ai, s4.x);
            float2 o1 = tc_out(__uint_as_float(v[16 * h + j + 1]), ai, s4.y);
            float2 o2 = tc_out(__uint_as_float(v[16 * h + j + 2]), ai, s4.z);
            float2 o3 = tc_out(__uint_as_float(v[16 * h + j + 3]), ai, s4.w);
            if (drow) {
              o0 = gadd_elem(o0, drow[cc]);
              o1 = gadd_elem(o1, drow[cc + 1]);
              o2 = gadd_elem(o2, drow[cc + 2]);
              o3 = gadd_elem(o3, drow[cc + 3]);
            }
            // [32 rows][16 cols] complex64, 128B-swizzled: 16-byte chunk c of row r at c ^ (r & 7)
            const uint32_t rb = sbuf + (uint32_t)lane * 128;
            // staging stores without a memory clobber: the column-scale / bias loads of the
            // following columns may be hoisted past them (with it, each waited serially)
            st_shared_v4_staging(rb + ((((j >> 1) + 0) ^ (lane & 7)) << 4), __float_as_uint(o0.x),
                                 __float_as_uint(o0.y), __float_as_uint(o1.x), __float_as_uint(o1.y));
            st_shared_v4_staging(rb + ((((j >> 1) + 1) ^ (lane & 7)) << 4), __float_as_uint(o2.x),
                                 __float_as_uint(o2.y), __float_as_uint(o3.x), __float_as_uint(o3.y));
            const uint32_t c0 = __float_as_uint(fmaxf(o0.x, 0.0f));
            const uint32_t c1 = __float_as_uint(fmaxf(o1.x, 0.0f));
            const uint32_t c2 = __float_as_uint(fmaxf(o2.x, 0.0f));
            const uint32_t c3 = __float_as_uint(fmaxf(o3.x, 0.0f));
            rmax = max(rmax, max(max(c0, c1), max(c2, c3)));
            if (emit.col) {
              const uint32_t m0 = __reduce_max_sync(0xffffffffu, c0);
              const uint32_t m1 = __reduce_max_sync(0xffffffffu, c1);
              const uint32_t m2 = __reduce_max_sync(0xffffffffu, c2);
              const uint32_t m3 = __reduce_max_sync(0xffffffffu, c3);
              if (lane == 0) {
                unsigned int* ce = reinterpret_cast<unsigned int*>(emit.col + b * emit.col_stride +
                                                                   pcol0 + cc);
                atomicMax(ce, m0);
                atomicMax(ce + 1, m1);
                atomicMax(ce + 2, m2);
                atomicMax(ce + 3, m3);
              }
            }
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (kFuse)  // the output streams out: evict_first keeps L2 for the scale-pass lines
              tma_store_3d_hint(&mapC, sbuf, pcol0 + col + 16 * h, wrow0, (int)b, pol_out);
            else
              tma_store_3d(&mapC, sbuf, pcol0 + col + 16 * h, wrow0, (int)b);
          }
        }
      }
      if (emit.row)
        atomicMax(reinterpret_cast<unsigned int*>(emit.row + b * emit.row_stride + grow), rmax);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_rank(acc_empty0 + buf * 8, 0);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's smem and barriers stay alive until the pair is done
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

// GOOM_TC_DEBUG (profiling only; results invalid unless noted): +64 one scale stage per main
// stage in the fused-scale pair kernel instead of GOOM_TC_LATE's lateness (results valid);
// 1 no transform, 2 no MMA, 3 no loads
// and no transform, 4 no loads, 5 loads only (no transform / MMA), 7 as 5 without the
// epilogue body, 8 MMA only (no loads / transform / epilogue body), 9 epilogue only
int tc_debug() {
  static int v = [] {
    const char* e = getenv("GOOM_TC_DEBUG");
    return e ? atoi(e) : 0;
  }();
  return v;
}
int late_factor() {
  static const int v = fuse_lateness("GOOM_TC_LATE", 8) & 15;
  return v;
}

template <bool kFuse>
int query_clusters() {
  return [] {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * 74);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Tc2Cfg<kFuse>::kSmem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, lmme_tc2_kernel<kFuse>, &cfg) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = num_sms() / 2;
    }
    return n;
  }();
}
template <bool kFuse>
int max_clusters() {  // per device (abi.cu per_device_value)
  return per_device_value((const void*)lmme_tc2_kernel<kFuse>, &query_clusters<kFuse>);
}

// GOOM_TC2_FUSE: 1 always reduce the scales in-kernel when the caller gives none, 0 never
// (pre-pass), unset: in-kernel when every A row block and B column block is read by exactly
// one pair tile (n == m == 256: the HBM-bound config-2 shape), so the reduction adds no
// second read of anything
int fuse_mode() {
  static int v = [] {
    const char* e = getenv("GOOM_TC2_FUSE");
    return e ? atoi(e) : -1;
  }();
  return v;
}

}  // namespace

bool lmme_tc2_eligible(int n, int k, int m) {
  return n > 0 && k > 0 && m > 0 && n % 256 == 0 && m % 256 == 0 && k % BK == 0;
}

bool lmme_tc2_fuse_scales(int n, int k, int m) {
  if (!lmme_tc2_eligible(n, k, m) || k < 128) return false;  // >= 8 K-blocks per tile (slot reuse)
  const int f = fuse_mode();
  return f == 1 || (f < 0 && n == 256 && m == 256);
}

template <bool kFuse>
int lmme_tc2_run(const LmmeProblem& p, cudaStream_t s);

int lmme_tc2(const LmmeProblem& p, cudaStream_t s) {
  if (!lmme_tc2_eligible(p.n, p.k, p.m)) return GOOM_EUNSUPPORTED;
  if (!p.rowA.ptr || !p.colB.ptr) {
    if (!lmme_tc2_fuse_scales(p.n, p.k, p.m)) return GOOM_EUNSUPPORTED;
    return lmme_tc2_run<true>(p, s);
  }
  return lmme_tc2_run<false>(p, s);
}

template <bool kFuse>
int lmme_tc2_run(const LmmeProblem& p, cudaStream_t s) {
  constexpr int kSmem = Tc2Cfg<kFuse>::kSmem;
  // TMA: 16-byte aligned bases and even matrix strides; epilogue: float4 column-scale
  // loads and 16-byte output stores
  if (((reinterpret_cast<uintptr_t>(p.A.ptr) | reinterpret_cast<uintptr_t>(p.B.ptr) |
        reinterpret_cast<uintptr_t>(p.C) | reinterpret_cast<uintptr_t>(p.colB.ptr)) & 15) ||
      ((p.A.stride | p.B.stride | p.strideC) & 1) || (p.colB.stride & 3))
    return GOOM_EUNSUPPORTED;
  GOOM_TRY(smem_attr((const void*)lmme_tc2_kernel<kFuse>, kSmem, "lmme_tc2 smem attribute"));
  alignas(64) CUtensorMap mapA, mapB;
  int64_t mats, mstride;
  // A: (k, n, matrix) complex64 moved as int64; box 16 k x 128 rows (one CTA's half)
  mats_of(p.A, p.batch, p.n, p.k, mats, mstride);
  {
    cuuint64_t dims[3] = {(cuuint64_t)p.k, (cuuint64_t)p.n, (cuuint64_t)mats};
    cuuint64_t strides[2] = {(cuuint64_t)p.k * 8, (cuuint64_t)mstride * 8};
    cuuint32_t box[3] = {BK, kRowsCta, 1};
    GOOM_TRY(encode(&mapA, p.A, 3, dims, strides, box));
  }
  // B: (8 cols, k_hi = k/4 [4 rows], k_lo [1 row], m/8 column groups, matrix);
  // box 8 x 4 x 4 x 16 x 1 -> smem [group][k_lo][k_hi][8]: row s holds k = 4 (s % 4) + s / 4
  mats_of(p.B, p.batch, p.k, p.m, mats, mstride);
  {
    cuuint64_t dims[5] = {8, (cuuint64_t)p.k / 4, 4, (cuuint64_t)(p.m / 8), (cuuint64_t)mats};
    cuuint64_t strides[4] = {(cuuint64_t)p.m * 8 * 4, (cuuint64_t)p.m * 8, 64,
                             (cuuint64_t)mstride * 8};
    cuuint32_t box[5] = {8, 4, 4, kPairN / 2 / 8, 1};
    GOOM_TRY(encode(&mapB, p.B, 5, dims, strides, box));
  }
  // C: (m, n, batch) complex64 as int64, box 16 cols x 32 rows, 128B swizzle (epilogue store)
  alignas(64) CUtensorMap mapC;
  {
    const int64_t cb = p.strideC == 0 ? 1 : p.batch;
    const int64_t cs = p.strideC == 0 ? (int64_t)p.n * p.m : p.strideC;
    cuuint64_t dims[3] = {(cuuint64_t)p.m, (cuuint64_t)p.n, (cuuint64_t)cb};
    cuuint64_t strides[2] = {(cuuint64_t)p.m * 8, (cuuint64_t)cs * 8};
    cuuint32_t box[3] = {16, 32, 1};
    GOOM_TRY(encode(&mapC, Operand{p.C, 0, 1}, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B));
  }
  PairGrid pg;
  pg.nct = p.m / kPairN;
  pg.nrt = p.n / 256;
  pg.tiles = p.batch * pg.nct * pg.nrt;
  const int64_t mc = max_clusters<kFuse>();
  const int64_t clusters = pg.tiles < mc ? pg.tiles : mc;
  Emit emit{p.emitRow, p.emitRowStride, p.emitCol, p.emitColStride};

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * clusters));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, lmme_tc2_kernel<kFuse>, mapA, mapB, mapC, p.A, p.B, p.D, p.rowA, p.colB, p.C,
                     p.strideC, pg, p.k, p.m, p.noncanon, emit,
      tc_debug() | (fit_lateness(late_factor(), p.k / BK) << 8));
  GOOM_CHECK_LAUNCH("lmme_tc2_kernel");
  return GOOM_OK;
}

}  // namespace goom
