// FP32 SIMT LMME kernels (Eq. 10-12, restating core._lmme_arrays core.py:242-261).
//
//  * lmme_small: one warp per product for n, k, m <= 32. The warp loads both
//    operands once into registers (lane l owns column l), reduces the clamped
//    row / column scales with shuffles, writes sign*exp(x - scale) to shared
//    memory and accumulates column l of the product in FP32 registers. Used by
//    the small-d scan paths (d = 8..32) and for d x 1 bias products.
//  * lmme_tiled: 64x64x16 shared-memory tiles, 256 threads x (4x4) outputs,
//    register-prefetched next K-tile; the scales come from the pre-pass. General
//    fallback for shapes the tcgen05 kernel does not tile (d = 33..127, ragged).
//
// Epilogue in registers: C = (log|I| + a_i) + b_j, sign(I) -> canonical
// complex64; optionally fused with the bias-slot gadd of combine_affine.
#include "goom_internal.cuh"

namespace goom {

namespace {

__device__ __forceinline__ float2 lmme_epilogue(float acc, float a, float b) {
  // (log|I| + a) + b in this order, as numpy evaluates core.py:259
  float lg = __fadd_rn(__fadd_rn(logf(fabsf(acc)), a), b);
  return make_float2(lg, acc < 0.0f ? kPi : 0.0f);
}

// ------------------------------------------------------------------------------
constexpr int kSmallWarps = 4;
constexpr int kSmallPitch = 33;

__global__ void __launch_bounds__(kSmallWarps * 32)
    lmme_small_kernel(Operand A, Operand B, Operand D, float2* __restrict__ C, int64_t strideC,
                      int64_t batch, int n, int k, int m) {
  __shared__ float sA[kSmallWarps][32 * kSmallPitch];  // [i][kk]
  __shared__ float sB[kSmallWarps][32 * kSmallPitch];  // [kk][j]
  const int wid = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t b = blockIdx.x * (int64_t)kSmallWarps + wid;
  if (b >= batch) return;
  const float2* a = A.at(b);
  const float2* bm = B.at(b);
  float* tA = sA[wid];
  float* tB = sB[wid];

  // column scale of B: lane j scans column j
  float bj = kNegInf;
  if (lane < m)
    for (int kk = 0; kk < k; ++kk) bj = fmaxf(bj, bm[kk * m + lane].x);
  bj = fmaxf(bj, 0.0f);
  for (int kk = 0; kk < k; ++kk) {
    float v = 0.0f;
    if (lane < m) {
      float2 z = bm[kk * m + lane];
      v = goom_sign(z.y) * expf(z.x - bj);
    }
    tB[kk * kSmallPitch + lane] = v;
  }
  // row scales of A: row i is read across lanes (lane = kk)
  float my_ai = 0.0f;  // lane i keeps a_i for the epilogue
  for (int i = 0; i < n; ++i) {
    float2 z = lane < k ? a[i * k + lane] : make_float2(kNegInf, 0.0f);
    float ai = fmaxf(warp_max(z.x), 0.0f);
    if (lane == i) my_ai = ai;
    tA[i * kSmallPitch + lane] = lane < k ? goom_sign(z.y) * expf(z.x - ai) : 0.0f;
  }
  __syncwarp();

  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = 0.0f;
  for (int kk = 0; kk < k; ++kk) {
    float bv = tB[kk * kSmallPitch + lane];
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < n) acc[i] = fmaf(tA[i * kSmallPitch + kk], bv, acc[i]);
  }
  float2* c = C + b * strideC;
  const float2* dd = D.ptr ? D.at(b) : nullptr;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i < n) {
      float ai = __shfl_sync(0xffffffffu, my_ai, i);
      if (lane < m) {
        float2 r = lmme_epilogue(acc[i], ai, bj);
        if (dd) r = gadd_elem(r, dd[i * m + lane]);
        c[i * m + lane] = r;
      }
    }
  }
}

// ------------------------------------------------------------------------------
constexpr int TM = 64, TN = 64, TK = 16, TPAD = 4;

__global__ void __launch_bounds__(256)
    lmme_tiled_kernel(Operand A, Operand B, Operand D, Scales rowA, Scales colB,
                      float2* __restrict__ C, int64_t strideC, int64_t b_base, int n, int k,
                      int m) {
  __shared__ __align__(16) float sA[TK][TM + TPAD];  // transposed: [kk][row]
  __shared__ __align__(16) float sB[TK][TN + TPAD];  // [kk][col]
  const int64_t b = b_base + blockIdx.z;
  const int row0 = blockIdx.y * TM;
  const int col0 = blockIdx.x * TN;
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const float2* a = A.at(b);
  const float2* bm = B.at(b);
  const float* ra = rowA.at(b);
  const float* cb = colB.at(b);

  // loader mapping: A tile 64 rows x 16 kk -> thread: row = tid/4, kk = (tid%4)*4 .. +4
  const int la_r = tid >> 2, la_k = (tid & 3) * 4;
  // B tile 16 kk x 64 cols -> thread: kk = tid/16, col = (tid%16)*4 .. +4
  const int lb_k = tid >> 4, lb_c = (tid & 15) * 4;
  const float a_scale = (row0 + la_r < n) ? ra[row0 + la_r] : 0.0f;
  float b_scale[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) b_scale[j] = (col0 + lb_c + j < m) ? cb[col0 + lb_c + j] : 0.0f;

  float2 ra_buf[4], rb_buf[4];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int r = row0 + la_r, kk = k0 + la_k + j;
      ra_buf[j] = (r < n && kk < k) ? a[(int64_t)r * k + kk] : make_float2(kNegInf, 0.0f);
      int kb = k0 + lb_k, c = col0 + lb_c + j;
      rb_buf[j] = (kb < k && c < m) ? bm[(int64_t)kb * m + c] : make_float2(kNegInf, 0.0f);
    }
  };

  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

  fetch(0);
  for (int k0 = 0; k0 < k; k0 += TK) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      sA[la_k + j][la_r] = goom_sign(ra_buf[j].y) * expf(ra_buf[j].x - a_scale);
      sB[lb_k][lb_c + j] = goom_sign(rb_buf[j].y) * expf(rb_buf[j].x - b_scale[j]);
    }
    __syncthreads();
    if (k0 + TK < k) fetch(k0 + TK);
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float4 av = *reinterpret_cast<const float4*>(&sA[kk][ty * 4]);
      float4 bv = *reinterpret_cast<const float4*>(&sB[kk][tx * 4]);
      float ar[4] = {av.x, av.y, av.z, av.w};
      float br[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(ar[i], br[j], acc[i][j]);
    }
    __syncthreads();
  }

  float2* c = C + b * strideC;
  const float2* dd = D.ptr ? D.at(b) : nullptr;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int r = row0 + ty * 4 + i;
    if (r >= n) continue;
    float ai = ra[r];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int cc = col0 + tx * 4 + j;
      if (cc >= m) continue;
      float2 o = lmme_epilogue(acc[i][j], ai, cb[cc]);
      if (dd) o = gadd_elem(o, dd[(int64_t)r * m + cc]);
      c[(int64_t)r * m + cc] = o;
    }
  }
}

}  // namespace

int lmme_simt_small(const LmmeProblem& p, cudaStream_t s) {
  unsigned grid = (unsigned)((p.batch + kSmallWarps - 1) / kSmallWarps);
  lmme_small_kernel<<<grid, kSmallWarps * 32, 0, s>>>(p.A, p.B, p.D, p.C, p.strideC, p.batch, p.n,
                                                     p.k, p.m);
  GOOM_CHECK_LAUNCH("lmme_small_kernel");
  return GOOM_OK;
}

int lmme_simt_tiled(const LmmeProblem& p, cudaStream_t s) {
  // grid.z carries the batch (<= 65535 per launch); split larger batches
  const int64_t zmax = 65535;
  for (int64_t b0 = 0; b0 < p.batch; b0 += zmax) {
    int64_t nb = p.batch - b0 < zmax ? p.batch - b0 : zmax;
    dim3 grid(ceil_div(p.m, TN), ceil_div(p.n, TM), (unsigned)nb);
    lmme_tiled_kernel<<<grid, 256, 0, s>>>(p.A, p.B, p.D, p.rowA, p.colB, p.C, p.strideC, b0,
                                           p.n, p.k, p.m);
    GOOM_CHECK_LAUNCH("lmme_tiled_kernel");
  }
  return GOOM_OK;
}

}  // namespace goom
