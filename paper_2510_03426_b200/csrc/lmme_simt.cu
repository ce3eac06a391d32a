// SIMT LMME kernels (Eq. 10-12, restating core._lmme_arrays core.py:242-261),
// generic over the backing precision (FP32 for complex64, FP64 for complex128).
//
//  * lmme_small: one warp per product for n, k, m <= 32. Lane l owns column l:
//    the warp reduces the clamped row / column scales with shuffles, writes
//    sign*exp(x - scale) to shared memory and accumulates column l of the
//    product in registers. Used by the small-d scan paths and d x 1 products.
//  * lmme_tiled: 64x64x16 shared-memory tiles, 256 threads x (4x4) outputs,
//    register-prefetched next K-tile; scales come from the pre-pass. Serves
//    complex128 and the complex64 shapes the tcgen05 kernel does not tile.
// Each output accumulates its dot product in ascending k with one FMA per
// term, so every kernel here (and the CTA-level LMME of the selective walk)
// returns bitwise-identical results for the same operands.
// Epilogue in registers: C = (log|I| + a_i) + b_j, sign(I) -> canonical GOOMs;
// optionally fused with the bias-slot gadd of combine_affine.
#include "goom_internal.cuh"

namespace goom {

namespace {

template <class R> constexpr int small_warps() { return sizeof(R) == 4 ? 4 : 2; }
constexpr int kSmallPitch = 33;

template <class R>
__global__ void __launch_bounds__(128)
    lmme_small_kernel(OperandT<Cx<R>> A, OperandT<Cx<R>> B, OperandT<Cx<R>> D,
                      Cx<R>* __restrict__ C, int64_t strideC, int64_t batch, int n, int k,
                      int m) {
  __shared__ R sA[small_warps<R>()][32 * kSmallPitch];  // [i][kk]
  __shared__ R sB[small_warps<R>()][32 * kSmallPitch];  // [kk][j]
  const int wid = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t b = blockIdx.x * (int64_t)small_warps<R>() + wid;
  if (b >= batch) return;
  const Cx<R>* a = A.at(b);
  const Cx<R>* bm = B.at(b);
  R* tA = sA[wid];
  R* tB = sB[wid];

  // column scale of B: lane j scans column j
  R bj = R(-INFINITY);
  if (lane < m)
    for (int kk = 0; kk < k; ++kk) bj = gmax(bj, bm[kk * m + lane].x);
  bj = gmax(bj, R(0));
  for (int kk = 0; kk < k; ++kk) {
    R v = R(0);
    if (lane < m) {
      Cx<R> z = bm[kk * m + lane];
      v = goom_sign_t<R>(z.y) * gexp(z.x - bj);
    }
    tB[kk * kSmallPitch + lane] = v;
  }
  // row scales of A: row i is read across lanes (lane = kk)
  R my_ai = R(0);  // lane i keeps a_i for the epilogue
  for (int i = 0; i < n; ++i) {
    Cx<R> z = lane < k ? a[i * k + lane] : cx<R>(R(-INFINITY), R(0));
    R ai = gmax(warp_max_t(z.x), R(0));
    if (lane == i) my_ai = ai;
    tA[i * kSmallPitch + lane] = lane < k ? goom_sign_t<R>(z.y) * gexp(z.x - ai) : R(0);
  }
  __syncwarp();

  R acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = R(0);
  for (int kk = 0; kk < k; ++kk) {
    R bv = tB[kk * kSmallPitch + lane];
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < n) acc[i] = gfma(tA[i * kSmallPitch + kk], bv, acc[i]);
  }
  Cx<R>* c = C + b * strideC;
  const Cx<R>* dd = D.ptr ? D.at(b) : nullptr;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i < n) {
      R ai = __shfl_sync(0xffffffffu, my_ai, i);
      if (lane < m) {
        Cx<R> r = lmme_out<R>(acc[i], ai, bj);
        if (dd) r = gadd_elem_t<R>(r, dd[i * m + lane]);
        c[i * m + lane] = r;
      }
    }
  }
}

// four consecutive values from 16-byte aligned shared memory in one or two vector loads
__device__ __forceinline__ void lds4(const float* p, float (&v)[4]) {
  const float4 x = *reinterpret_cast<const float4*>(p);
  v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
}
__device__ __forceinline__ void lds4(const double* p, double (&v)[4]) {
  const double2 x = *reinterpret_cast<const double2*>(p);
  const double2 y = *reinterpret_cast<const double2*>(p + 2);
  v[0] = x.x, v[1] = x.y, v[2] = y.x, v[3] = y.y;
}

// ------------------------------------------------------------------------------
constexpr int TM = 64, TN = 64, TK = 16, TPAD = 4;

template <class R>
__global__ void __launch_bounds__(256)
    lmme_tiled_kernel(OperandT<Cx<R>> A, OperandT<Cx<R>> B, OperandT<Cx<R>> D, ScalesT<R> rowA,
                      ScalesT<R> colB, Cx<R>* __restrict__ C, int64_t strideC, int64_t b_base,
                      int n, int k, int m) {
  __shared__ __align__(16) R sA[TK][TM + TPAD];  // transposed: [kk][row]
  __shared__ __align__(16) R sB[TK][TN + TPAD];  // [kk][col]
  const int64_t b = b_base + blockIdx.z;
  const int row0 = blockIdx.y * TM;
  const int col0 = blockIdx.x * TN;
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const Cx<R>* a = A.at(b);
  const Cx<R>* bm = B.at(b);
  const R* ra = rowA.at(b);
  const R* cb = colB.at(b);

  // loader mapping: A tile 64 rows x 16 kk -> thread: row = tid/4, kk = (tid%4)*4 .. +4
  const int la_r = tid >> 2, la_k = (tid & 3) * 4;
  // B tile 16 kk x 64 cols -> thread: kk = tid/16, col = (tid%16)*4 .. +4
  const int lb_k = tid >> 4, lb_c = (tid & 15) * 4;
  const R a_scale = (row0 + la_r < n) ? ra[row0 + la_r] : R(0);
  R b_scale[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) b_scale[j] = (col0 + lb_c + j < m) ? cb[col0 + lb_c + j] : R(0);

  Cx<R> ra_buf[4], rb_buf[4];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int r = row0 + la_r, kk = k0 + la_k + j;
      ra_buf[j] = (r < n && kk < k) ? a[(int64_t)r * k + kk] : cx<R>(R(-INFINITY), R(0));
      int kb = k0 + lb_k, c = col0 + lb_c + j;
      rb_buf[j] = (kb < k && c < m) ? bm[(int64_t)kb * m + c] : cx<R>(R(-INFINITY), R(0));
    }
  };

  R acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = R(0);

  fetch(0);
  for (int k0 = 0; k0 < k; k0 += TK) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      sA[la_k + j][la_r] = goom_sign_t<R>(ra_buf[j].y) * gexp(ra_buf[j].x - a_scale);
      sB[lb_k][lb_c + j] = goom_sign_t<R>(rb_buf[j].y) * gexp(rb_buf[j].x - b_scale[j]);
    }
    __syncthreads();
    if (k0 + TK < k) fetch(k0 + TK);
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      R ar[4], br[4];
      lds4(&sA[kk][ty * 4], ar);
      lds4(&sB[kk][tx * 4], br);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = gfma(ar[i], br[j], acc[i][j]);
    }
    __syncthreads();
  }

  Cx<R>* c = C + b * strideC;
  const Cx<R>* dd = D.ptr ? D.at(b) : nullptr;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int r = row0 + ty * 4 + i;
    if (r >= n) continue;
    R ai = ra[r];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int cc = col0 + tx * 4 + j;
      if (cc >= m) continue;
      Cx<R> o = lmme_out<R>(acc[i][j], ai, cb[cc]);
      if (dd) o = gadd_elem_t<R>(o, dd[(int64_t)r * m + cc]);
      c[(int64_t)r * m + cc] = o;
    }
  }
}

// ------------------------------------------------------------------------------
// lmme_whole: one CTA per product for n, k, m <= 64 with the scales fused: the CTA reads
// A and B once (coalesced) into shared memory as log-magnitude and sign planes, reduces
// the clamped row / column maxima there, exponentiates in place into the tiled kernel's
// [kk][row] / [kk][col] layout and runs the same 4 x 4-per-thread GEMM (ascending kk, one
// FMA per term) and epilogue — bitwise equal to scale pre-pass + lmme_tiled, with one
// HBM pass (24 B per element for complex64) instead of three reads.
constexpr int kWholePitch = 64 + TPAD;

template <class R>
__global__ void __launch_bounds__(256)
    lmme_whole_kernel(OperandT<Cx<R>> A, OperandT<Cx<R>> B, OperandT<Cx<R>> D,
                      Cx<R>* __restrict__ C, int64_t strideC, int64_t b_base, int n, int k,
                      int m) {
  extern __shared__ __align__(16) unsigned char whole_smem[];
  R* sA = reinterpret_cast<R*>(whole_smem);   // [kk][row]: log, then sign * exp(log - a)
  R* sB = sA + 64 * kWholePitch;              // [kk][col]
  R* sc = sB + 64 * kWholePitch;              // [0, 64) a_i, [64, 128) b_j
  signed char* gA = reinterpret_cast<signed char*>(sc + 128);  // signs (+1 / -1), same layouts
  signed char* gB = gA + 64 * kWholePitch;
  const int64_t b = b_base + blockIdx.x;
  const Cx<R>* a = A.at(b);
  const Cx<R>* bm = B.at(b);
  const int tid = threadIdx.x;
  for (int e = tid; e < n * k; e += 256) {  // coalesced over A's row-major storage
    const int i = e / k, kk = e % k;
    const Cx<R> z = a[e];
    sA[kk * kWholePitch + i] = z.x;
    gA[kk * kWholePitch + i] = goom_sign_t<R>(z.y) < R(0) ? -1 : 1;
  }
  for (int e = tid; e < k * m; e += 256) {
    const int kk = e / m, j = e % m;
    const Cx<R> z = bm[e];
    sB[kk * kWholePitch + j] = z.x;
    gB[kk * kWholePitch + j] = goom_sign_t<R>(z.y) < R(0) ? -1 : 1;
  }
  __syncthreads();
  if (tid < 64) {  // clamped row maxima of A (max is exact: any order)
    R v = R(-INFINITY);
    if (tid < n)
      for (int kk = 0; kk < k; ++kk) v = gmax(v, sA[kk * kWholePitch + tid]);
    sc[tid] = gmax(v, R(0));
  } else if (tid < 128) {  // clamped column maxima of B
    const int j = tid - 64;
    R v = R(-INFINITY);
    if (j < m)
      for (int kk = 0; kk < k; ++kk) v = gmax(v, sB[kk * kWholePitch + j]);
    sc[tid] = gmax(v, R(0));
  }
  __syncthreads();
  for (int e = tid; e < 64 * k; e += 256) {
    const int kk = e >> 6, c = e & 63;
    const int o = kk * kWholePitch + c;
    sA[o] = c < n ? R(gA[o]) * gexp(sA[o] - sc[c]) : R(0);
    sB[o] = c < m ? R(gB[o]) * gexp(sB[o] - sc[64 + c]) : R(0);
  }
  __syncthreads();
  const int tx = tid & 15, ty = tid >> 4;
  R acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = R(0);
  for (int kk = 0; kk < k; ++kk) {
    R ar[4], br[4];
    lds4(&sA[kk * kWholePitch + ty * 4], ar);
    lds4(&sB[kk * kWholePitch + tx * 4], br);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = gfma(ar[i], br[j], acc[i][j]);
  }
  Cx<R>* c = C + b * strideC;
  const Cx<R>* dd = D.ptr ? D.at(b) : nullptr;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = ty * 4 + i;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cc = tx * 4 + j;
      if (cc >= m) continue;
      Cx<R> o = lmme_out<R>(acc[i][j], sc[r], sc[64 + cc]);
      if (dd) o = gadd_elem_t<R>(o, dd[(int64_t)r * m + cc]);
      c[(int64_t)r * m + cc] = o;
    }
  }
}

// n = k = m = 64 complex64 with 16-byte aligned operands (the config-2 d = 64 shape): the
// whole-product kernel with all of a thread's operand loads issued up front (16 x 16 B in
// flight, where the generic loop above keeps one 8 B load per thread), the row scales of A
// reduced by the warp that holds the row (shuffles), B's column scales through one 2 KB
// table, and A kept row-major so the k loop reads four k at a time per row. Accumulation
// order (ascending k, one FMA per term) and the epilogue are the generic kernel's, so the
// results are bitwise identical.
constexpr int kP64 = 68;

__device__ __forceinline__ float2 unit_pair(float4 z, float s0, float s1) {
  return make_float2(goom_sign_t<float>(z.y) * gexp(z.x - s0),
                     goom_sign_t<float>(z.w) * gexp(z.z - s1));
}

__global__ void __launch_bounds__(256, 3)
    lmme_whole64_kernel(OperandT<float2> A, OperandT<float2> B, OperandT<float2> D,
                        float2* __restrict__ C, int64_t strideC, int64_t b_base) {
  __shared__ __align__(16) float sA[64 * kP64];  // [i][kk]: sign * exp(log - a_i)
  __shared__ __align__(16) float sB[64 * kP64];  // [kk][j]: sign * exp(log - b_j)
  __shared__ __align__(16) float sRed[8][64];    // per-warp partial column maxima of B
  __shared__ float sc[128];                      // a_i, then b_j
  const int64_t b = b_base + blockIdx.x;
  const float4* a4 = reinterpret_cast<const float4*>(A.at(b));
  const float4* b4 = reinterpret_cast<const float4*>(B.at(b));
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // float4 q = tid + 256 r holds elements 2q, 2q + 1: row / k index w + 8 r, column 2 lane
  float4 ra[8], rb[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) ra[r] = __ldcs(a4 + tid + 256 * r);
#pragma unroll
  for (int r = 0; r < 8; ++r) rb[r] = __ldcs(b4 + tid + 256 * r);
#pragma unroll
  for (int r = 0; r < 8; ++r) {  // row w + 8 r of A lives in this warp
    float v = gmax(ra[r].x, ra[r].z);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = gmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    v = gmax(v, 0.f);
    if (lane == 0) sc[w + 8 * r] = v;
    *reinterpret_cast<float2*>(&sA[(w + 8 * r) * kP64 + 2 * lane]) = unit_pair(ra[r], v, v);
  }
  float c0 = -INFINITY, c1 = -INFINITY;
#pragma unroll
  for (int r = 0; r < 8; ++r) c0 = gmax(c0, rb[r].x), c1 = gmax(c1, rb[r].z);
  *reinterpret_cast<float2*>(&sRed[w][2 * lane]) = make_float2(c0, c1);
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const float2 p = *reinterpret_cast<const float2*>(&sRed[u][2 * lane]);
    c0 = gmax(c0, p.x), c1 = gmax(c1, p.y);
  }
  c0 = gmax(c0, 0.f), c1 = gmax(c1, 0.f);
  if (w == 0) sc[64 + 2 * lane] = c0, sc[65 + 2 * lane] = c1;
#pragma unroll
  for (int r = 0; r < 8; ++r)
    *reinterpret_cast<float2*>(&sB[(w + 8 * r) * kP64 + 2 * lane]) = unit_pair(rb[r], c0, c1);
  __syncthreads();
  const int tx = tid & 15, ty = tid >> 4;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 2
  for (int k0 = 0; k0 < 64; k0 += 4) {
    float ar[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) lds4(&sA[(ty * 4 + i) * kP64 + k0], ar[i]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float br[4];
      lds4(&sB[(k0 + q) * kP64 + tx * 4], br);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = gfma(ar[i][q], br[j], acc[i][j]);
    }
  }
  float2* c = C + b * strideC;
  const float2* dd = D.ptr ? D.at(b) : nullptr;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = ty * 4 + i;
    float2 o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = lmme_out<float>(acc[i][j], sc[r], sc[64 + tx * 4 + j]);
    if (dd) {
      const float4* d4 = reinterpret_cast<const float4*>(dd + r * 64 + tx * 4);
      const float4 d0 = d4[0], d1 = d4[1];
      o[0] = gadd_elem(o[0], make_float2(d0.x, d0.y));
      o[1] = gadd_elem(o[1], make_float2(d0.z, d0.w));
      o[2] = gadd_elem(o[2], make_float2(d1.x, d1.y));
      o[3] = gadd_elem(o[3], make_float2(d1.z, d1.w));
    }
    float4* c4 = reinterpret_cast<float4*>(c + r * 64 + tx * 4);
    c4[0] = make_float4(o[0].x, o[0].y, o[1].x, o[1].y);
    c4[1] = make_float4(o[2].x, o[2].y, o[3].x, o[3].y);
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

template <class R>
size_t lmme_whole_smem() {
  return (size_t)(2 * 64 * kWholePitch + 128) * sizeof(R) + 2 * 64 * kWholePitch;
}

template <class R>
int lmme_simt_whole(const LmmeProblemT<R>& p, cudaStream_t s) {
  if constexpr (sizeof(R) == 4) {
    const bool vec = p.n == 64 && p.k == 64 && p.m == 64 && aligned16(p.A.ptr) &&
                     aligned16(p.B.ptr) && aligned16(p.C) && p.A.stride % 2 == 0 &&
                     p.B.stride % 2 == 0 && p.strideC % 2 == 0 &&
                     (!p.D.ptr || (aligned16(p.D.ptr) && p.D.stride % 2 == 0));
    static const bool generic = [] {
      const char* e = std::getenv("GOOM_WHOLE64_GENERIC");
      return e && e[0] == '1';
    }();
    if (vec && !generic) {
      const int64_t gmax_ = 2147483647;
      for (int64_t b0 = 0; b0 < p.batch; b0 += gmax_) {
        const int64_t nb = p.batch - b0 < gmax_ ? p.batch - b0 : gmax_;
        lmme_whole64_kernel<<<(unsigned)nb, 256, 0, s>>>(p.A, p.B, p.D, p.C, p.strideC, b0);
        GOOM_CHECK_LAUNCH("lmme_whole64_kernel");
      }
      return GOOM_OK;
    }
  }
  const size_t smem = lmme_whole_smem<R>();
  GOOM_TRY(smem_attr((const void*)lmme_whole_kernel<R>, (int)smem, "lmme_whole smem attribute"));
  const int64_t gmax_ = 2147483647;
  for (int64_t b0 = 0; b0 < p.batch; b0 += gmax_) {
    const int64_t nb = p.batch - b0 < gmax_ ? p.batch - b0 : gmax_;
    lmme_whole_kernel<R><<<(unsigned)nb, 256, smem, s>>>(p.A, p.B, p.D, p.C, p.strideC, b0, p.n,
                                                         p.k, p.m);
    GOOM_CHECK_LAUNCH("lmme_whole_kernel");
  }
  return GOOM_OK;
}

template <class R>
int lmme_simt_small(const LmmeProblemT<R>& p, cudaStream_t s) {
  constexpr int W = small_warps<R>();
  unsigned grid = (unsigned)((p.batch + W - 1) / W);
  lmme_small_kernel<R><<<grid, W * 32, 0, s>>>(p.A, p.B, p.D, p.C, p.strideC, p.batch,
                                                        p.n, p.k, p.m);
  GOOM_CHECK_LAUNCH("lmme_small_kernel");
  return GOOM_OK;
}

template <class R>
int lmme_simt_tiled(const LmmeProblemT<R>& p, cudaStream_t s) {
  // grid.z carries the batch (<= 65535 per launch); larger batches launch in slices
  const int64_t zmax = 65535;
  for (int64_t b0 = 0; b0 < p.batch; b0 += zmax) {
    int64_t nb = p.batch - b0 < zmax ? p.batch - b0 : zmax;
    dim3 grid(ceil_div(p.m, TN), ceil_div(p.n, TM), (unsigned)nb);
    lmme_tiled_kernel<R><<<grid, 256, 0, s>>>(p.A, p.B, p.D, p.rowA, p.colB, p.C, p.strideC, b0,
                                              p.n, p.k, p.m);
    GOOM_CHECK_LAUNCH("lmme_tiled_kernel");
  }
  return GOOM_OK;
}

template int lmme_simt_small<float>(const LmmeProblemT<float>&, cudaStream_t);
template int lmme_simt_small<double>(const LmmeProblemT<double>&, cudaStream_t);
template int lmme_simt_whole<float>(const LmmeProblemT<float>&, cudaStream_t);
template int lmme_simt_whole<double>(const LmmeProblemT<double>&, cudaStream_t);
template int lmme_simt_tiled<float>(const LmmeProblemT<float>&, cudaStream_t);
template int lmme_simt_tiled<double>(const LmmeProblemT<double>&, cudaStream_t);

}  // namespace goom
