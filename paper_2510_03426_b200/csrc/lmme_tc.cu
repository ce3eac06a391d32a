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
//   warps 18..21  epilogue : tcgen05.ld the accumulator, (log|I| + a_i) + b_j and the
//                            sign in registers (log via lg2.approx: abs. error ~1e-7,
//                            below the FP32 ulp of the output), optional fused gadd,
//                            store, and optionally the clamped row / column maxima of the
//                            output (the next LMME's scales: no pre-pass over C).
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
constexpr int STAGES = 4;
constexpr int kXformWarps = 16;
constexpr int kEpiWarps = 4;                     // one per TMEM lane quadrant
constexpr int kThreads = 64 + (kXformWarps + kEpiWarps) * 32;  // loader, MMA, transform, epilogue
constexpr int kGroupBytes = 1024;                // 8 rows x 16 k complex64 == 2 x 512 B TF32

template <int BN>
struct Cfg {
  static constexpr int kGroupsA = BM / 8;
  static constexpr int kGroupsB = BN / 8;
  static constexpr int kBytesA = kGroupsA * kGroupBytes;
  static constexpr int kStage = (kGroupsA + kGroupsB) * kGroupBytes;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered FP32 accumulator
  static constexpr int kRing = STAGES * kStage;
  static constexpr int kOut = kRing + 256;  // epilogue staging: [4 warps][32 rows][32 cols]
  static constexpr int kSmem = kOut + kEpiWarps * 8192 + 1024;
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

struct TileGrid {
  int nct, nrt;       // column / row tiles per product
  int64_t b_base;     // first product of this launch
  int64_t tiles;      // tiles in this launch
  __device__ __forceinline__ void at(int64_t t, int64_t& b, int& row0, int& col0, int BN) const {
    const int ct = (int)(t % nct);
    const int64_t q = t / nct;
    row0 = (int)(q % nrt) * BM;
    col0 = ct * BN;
    b = b_base + q / nrt;
  }
};

struct Emit {
  float* row;   // row[b * row_stride + i]: clamped row maxima of C (atomicMax on the bits)
  int64_t row_stride;
  float* col;   // col[b * col_stride + j]
  int64_t col_stride;
};

// Persistent kernel: grid = min(tiles, SMs); tiles in row-major (product, row tile, column
// tile) order, so concurrently resident tiles share operand panels in L2.
template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    lmme_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ CUtensorMap mapB3, Operand A, Operand B, Operand D, Scales rowA, Scales colB,
                   float2* __restrict__ C, int64_t strideC, TileGrid grid, int n, int k, int m,
                   const int* __restrict__ noncanon, Emit emit, int debug) {
  using G = Cfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KB-align the ring while keeping the pointer's shared-space provenance
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + G::kRing);
  uint64_t* full = bars;                    // [STAGES] TMA landed (tx bytes)
  uint64_t* ready = bars + STAGES;          // [STAGES] operands transformed (16 warp arrivals)
  uint64_t* freed = bars + 2 * STAGES;      // [STAGES] MMAs of the stage retired (commit)
  uint64_t* acc_full = bars + 3 * STAGES;   // [2] accumulator buffer complete (commit)
  uint64_t* acc_empty = acc_full + 2;       // [2] epilogue drained the buffer (4 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nk = k / BK;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&ready[s]), kXformWarps);
      mbar_init(smem_u32(&freed[s]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&acc_full[i]), 1);
      mbar_init(smem_u32(&acc_empty[i]), kEpiWarps);
    }
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

  if (warp == 0) {
    // ------------------------------ loader ------------------------------
    if (lane == 0) {
      int64_t g = 0;  // K-blocks issued so far (ring position)
      for (int64_t t = blockIdx.x; t < grid.tiles; t += gridDim.x) {
        int64_t b;
        int row0, col0;
        grid.at(t, b, row0, col0, BN);
        const int ma = A.stride == 0 ? 0 : (int)(b / A.div);
        const int mb = B.stride == 0 ? 0 : (int)(b / B.div);
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = (int)(g % STAGES);
          mbar_wait(smem_u32(&freed[s]), (uint32_t)((g / STAGES) & 1) ^ 1u);
          const uint32_t bar = smem_u32(&full[s]);
          if (debug >= 3) {  // profiling aid: no loads
            mbar_arrive(bar);
            continue;
          }
          mbar_expect_tx(bar, G::kStage);
          const uint32_t dst = ring + s * G::kStage;
          const int k0 = kb * BK;
          tma_load_3d(dst, &mapA, k0, row0, ma, bar);                      // [128 rows][16 k]
          if (debug == 6)  /* profiling aid: B as one 2 KB-row box (layout wrong) */
            tma_load_3d(dst + G::kBytesA, &mapB3, col0, k0, mb, bar);
          else
            tma_load_4d(dst + G::kBytesA, &mapB, 0, k0, col0 / 8, mb, bar);  // [BN/8][16 k][8 cols]
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ------------------------------
    if (lane == 0) {
      constexpr uint32_t idesc = tf32_idesc(BM, BN);
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
          if (debug != 2 && debug < 5) {
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
          }
          mma_commit(smem_u32(&freed[s]));  // the stage returns to the loader when these retire
        }
        mma_commit(smem_u32(&acc_full[buf]));  // accumulator of this tile complete
      }
    }
    __syncwarp();
  } else if (warp < 2 + kXformWarps) {
    // ------------------------------ transform (in place, software-pipelined) ---------------
    const int xw = warp - 2;
    const bool canon = noncanon != nullptr && *noncanon == 0;
    const int r = lane >> 3, bn = lane & 7;
    int64_t t = blockIdx.x;
    float sa0 = 0.f, sa1 = 0.f, sb[2] = {0.f, 0.f};
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
  } else {
    // ------------------------------ epilogue ------------------------------
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = quad * 32 + lane;
    const uint32_t stage = ring + G::kOut + (uint32_t)(warp - 2 - kXformWarps) * 8192u;
    int lt = 0;
    for (int64_t t = blockIdx.x; t < grid.tiles; t += gridDim.x, ++lt) {
      int64_t b;
      int row0, col0;
      grid.at(t, b, row0, col0, BN);
      const int buf = lt & 1;
      mbar_wait(smem_u32(&acc_full[buf]), (uint32_t)((lt >> 1) & 1));
      tc_fence_after();
      const float ai = rowA.at(b)[row0 + row];
      const float* cb = colB.at(b) + col0;
      float2* cblk = C + b * strideC + (int64_t)(row0 + quad * 32) * m + col0;
      const float2* drow = D.ptr ? D.at(b) + (int64_t)(row0 + row) * m + col0 : nullptr;
      uint32_t rmax = 0;  // bits of max(log, 0): non-negative floats order like uints
#pragma unroll 1
      for (int col = 0; col < (debug == 7 ? 0 : BN); col += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * BN + col), v);
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          float2 o0 = tc_out(__uint_as_float(v[j]), ai, cb[col + j]);
          float2 o1 = tc_out(__uint_as_float(v[j + 1]), ai, cb[col + j + 1]);
          if (drow) {
            o0 = gadd_elem(o0, drow[col + j]);
            o1 = gadd_elem(o1, drow[col + j + 1]);
          }
          // row `lane`, 16-byte chunk j / 2, XOR-swizzled by the row: conflict-free both ways
          // (no memory clobber: the column-scale loads above may be hoisted past it)
          st_shared_v4_staging(stage + lane * 256 + ((((j >> 1) ^ lane) & 15) << 4),
                       __float_as_uint(o0.x), __float_as_uint(o0.y), __float_as_uint(o1.x),
                       __float_as_uint(o1.y));
          const uint32_t c0 = __float_as_uint(fmaxf(o0.x, 0.0f));
          const uint32_t c1 = __float_as_uint(fmaxf(o1.x, 0.0f));
          rmax = max(rmax, max(c0, c1));
          if (emit.col) {
            const uint32_t m0 = __reduce_max_sync(0xffffffffu, c0);
            const uint32_t m1 = __reduce_max_sync(0xffffffffu, c1);
            if (lane == 0) {
              unsigned int* cc =
                  reinterpret_cast<unsigned int*>(emit.col + b * emit.col_stride + col0 + col + j);
              atomicMax(cc, m0);
              atomicMax(cc + 1, m1);
            }
          }
        }
        __syncwarp();
        // copy-out: two full 256-byte row segments per instruction (coalesced), where a
        // lane-per-row store would touch 32 lines per instruction
#pragma unroll 4
        for (int it = 0; it < 16; ++it) {
          const int rr = 2 * it + (lane >> 4), c = lane & 15;
          const float4 o = ld_shared_v4(stage + rr * 256 + (((c ^ rr) & 15) << 4));
          if (debug != 8) *reinterpret_cast<float4*>(cblk + (int64_t)rr * m + col + 2 * c) = o;
        }
        __syncwarp();
      }
      if (emit.row)
        atomicMax(reinterpret_cast<unsigned int*>(emit.row + b * emit.row_stride + row0 + row), rmax);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&acc_empty[buf]));
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

// GOOM_TC_DEBUG (profiling only; results invalid): 1 skips the transform, 2 the MMAs,
// 3 the TMA loads and the transform, 4 the TMA loads, 5 transform and MMAs (TMA ring only),
// 6 as 5 with B loaded as full-width rows, 7 skips the epilogue, 8 its global stores
int tc_debug() {
  static int v = [] {
    const char* e = getenv("GOOM_TC_DEBUG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <int BN>
int launch_tc(const LmmeProblem& p, cudaStream_t s) {
  GOOM_TRY(smem_attr((const void*)lmme_tc_kernel<BN>, Cfg<BN>::kSmem, "lmme_tc smem attribute"));
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
  alignas(64) CUtensorMap mapB3;  // GOOM_TC_DEBUG=6 only: B as [16 k][BN] rows of BN*8 bytes
  {
    cuuint64_t dims[3] = {(cuuint64_t)p.m, (cuuint64_t)p.k, (cuuint64_t)mats};
    cuuint64_t strides[2] = {(cuuint64_t)p.m * 8, (cuuint64_t)mstride * 8};
    cuuint32_t box[3] = {BN, BK, 1};
    GOOM_TRY(encode(&mapB3, p.B, 3, dims, strides, box));
  }
  TileGrid tg;
  tg.nct = p.m / BN;
  tg.nrt = p.n / BM;
  tg.b_base = 0;
  tg.tiles = p.batch * tg.nct * tg.nrt;
  const int64_t sms = num_sms();
  const unsigned grid = (unsigned)(tg.tiles < sms ? tg.tiles : sms);
  Emit emit{p.emitRow, p.emitRowStride, p.emitCol, p.emitColStride};
  lmme_tc_kernel<BN><<<grid, kThreads, Cfg<BN>::kSmem, s>>>(
      mapA, mapB, mapB3, p.A, p.B, p.D, p.rowA, p.colB, p.C, p.strideC, tg, p.n, p.k, p.m, p.noncanon,
      emit, tc_debug());
  GOOM_CHECK_LAUNCH("lmme_tc_kernel");
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
  static const bool pairs = [] {
    const char* e = getenv("GOOM_TC2");
    return !(e && atoi(e) == 0);
  }();
  if (pairs && lmme_tc2_eligible(p.n, p.k, p.m)) {
    const int rc = lmme_tc2(p, s);
    if (rc != GOOM_EUNSUPPORTED) return rc;
  }
  if (p.m % 256 == 0) return launch_tc<256>(p, s);
  return launch_tc<128>(p, s);
}

}  // namespace goom
