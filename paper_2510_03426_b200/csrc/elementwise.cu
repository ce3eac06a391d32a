// Elementwise GOOM kernels: real<->GOOM maps, scaled export, signed LSE (gadd),
// column log-norms, and the LMME scale pre-pass (row / column maxima).
//
// All are HBM-bound streaming kernels (8 or 16 B per complex element plus the
// real side); grid-stride loops sized to a multiple of the SM count.
#include "goom_internal.cuh"

namespace goom {

namespace {

constexpr int kThreads = 256;

inline int stream_grid(int64_t n) {
  int64_t blocks = (n + kThreads - 1) / kThreads;
  int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  return blocks < 1 ? 1 : (int)blocks;
}

#define GRID_STRIDE(i, n)                                                                   \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n);                 \
       i += (int64_t)gridDim.x * blockDim.x)

template <class X, class R>
__global__ void from_real_kernel(const X* __restrict__ x, Cx<R>* __restrict__ out, int64_t n,
                                 X zero_log) {
  GRID_STRIDE(i, n) {
    X v = x[i];
    if (v == X(0)) {
      out[i] = cx<R>((R)zero_log, R(0));
    } else {
      out[i] = cx<R>((R)glog(fabs(v)), v < X(0) ? pi_of<R>() : R(0));
    }
  }
}

template <class R, class X>
__global__ void to_real_kernel(const Cx<R>* __restrict__ z, X* __restrict__ out, int64_t n) {
  GRID_STRIDE(i, n) {
    Cx<R> v = z[i];
    out[i] = (X)goom_sign_t<R>(v.y) * gexp((X)v.x);
  }
}

// one CTA per matrix: max log, then the shifted export (core.py:313-323)
template <class R>
__global__ void to_real_scaled_kernel(const Cx<R>* __restrict__ z, R* __restrict__ out,
                                      R* __restrict__ cvec, int64_t n) {
  const int64_t b = blockIdx.x;
  const Cx<R>* zb = z + b * n;
  R* ob = out + b * n;
  __shared__ R red[32];
  R m = R(-INFINITY);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = gmax(m, zb[i].x);
  m = warp_max_t(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    R v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : R(-INFINITY);
    v = warp_max_t(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  R c = red[0];
  if (c == R(-INFINITY) || n == 0) c = R(0);
  if (threadIdx.x == 0) cvec[b] = c;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    Cx<R> v = zb[i];
    ob[i] = goom_sign_t<R>(v.y) * gexp(add_rn(sub_rn(v.x, c), R(2)));
  }
}

// SSM state export (ssm.py:84-98 on the chunked scan's output, no permuted copy): X is the
// state-assembly LMME's (H L, d, S nC) panels — state (h, s, t = cc L + i) is column
// s nC + cc of matrix h L + i. A CTA stages 32 columns x d rows (coalesced, padded against
// bank conflicts), then each warp takes whole states: c = max log (0 if none), and writes
// log, sign and sign * exp(log - c + 2) as contiguous d-vectors of the (H, S, T, d) outputs.
constexpr int kExportCols = 32;
__global__ void __launch_bounds__(256)
    ssm_export_kernel(const double2* __restrict__ X, int64_t L, int d, int64_t S, int64_t nC,
                      int64_t T, double* __restrict__ sl, double* __restrict__ ss,
                      double* __restrict__ cvec, double* __restrict__ z, int reverse,
                      const double* __restrict__ kshift, int64_t hi0) {
  __shared__ double2 tile[64][kExportCols + 1];
  const int64_t hi = hi0 + blockIdx.y, N = S * nC;  // (head, step) slice: grid.y <= 65535
  const int64_t h = hi / L, i = hi % L;
  const int64_t n0 = (int64_t)blockIdx.x * kExportCols;
  const int ncols = (int)(N - n0 < kExportCols ? N - n0 : kExportCols);
  const double2* xb = X + hi * d * N + n0;
  for (int e = threadIdx.x; e < d * kExportCols; e += 256) {
    const int r = e / kExportCols, j = e % kExportCols;
    if (j < ncols) tile[r][j] = xb[(int64_t)r * N + j];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int j = w; j < ncols; j += 8) {
    const int64_t n = n0 + j, s = n / nC, t = (n % nC) * L + i;
    if (t >= T) continue;
    double m = -INFINITY;
    for (int r = lane; r < d; r += 32) m = gmax(m, tile[r][j].x);
    m = warp_max_t(m);
    const double c = m == -INFINITY ? 0.0 : m;
    const int64_t o = ((h * S + s) * T + (reverse ? T - 1 - t : t)) * d;
    const double k = kshift ? kshift[h * S + s] : 0.0;
    if (lane == 0 && cvec) cvec[o / d] = c;
    for (int r = lane; r < d; r += 32) {
      const double2 v = tile[r][j];
      const double sg = cos(v.y) < 0.0 ? -1.0 : 1.0;
      sl[o + r] = kshift ? sub_rn(v.x, k) : v.x;
      ss[o + r] = sg;
      if (z) z[o + r] = sg * gexp(add_rn(sub_rn(v.x, c), 2.0));
    }
  }
}

// SSM backward source term, one warp per state (d <= 64: lane j holds elements j, j + 32)
__global__ void ssm_adjoint_source_kernel(const double* __restrict__ sl,
                                          const double* __restrict__ ss,
                                          const double* __restrict__ cvec,
                                          const double* __restrict__ gz, int64_t n, int d,
                                          double* __restrict__ h, double* __restrict__ z) {
  const int lane = threadIdx.x & 31;
  const int64_t st = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (st >= n) return;
  const int64_t o = st * d;
  const double c = cvec[st];
  double zv[2], gv[2], lv[2], sv[2];
  double m = -INFINITY, dot = 0.0;
  int im = 1 << 30;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = lane + 32 * q;
    if (j < d) {
      lv[q] = sl[o + j];
      sv[q] = ss[o + j];
      gv[q] = gz[o + j];
      zv[q] = sv[q] * exp(add_rn(sub_rn(lv[q], c), 2.0));
      dot = fma(gv[q], zv[q], dot);
      if (lv[q] > m) {  // first index of the maximum
        m = lv[q];
        im = j;
      }
    } else {
      lv[q] = sv[q] = gv[q] = zv[q] = 0.0;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double m2 = __shfl_xor_sync(0xffffffffu, m, off);
    const int i2 = __shfl_xor_sync(0xffffffffu, im, off);
    if (m2 > m || (m2 == m && i2 < im)) {
      m = m2;
      im = i2;
    }
    dot += __shfl_xor_sync(0xffffffffu, dot, off);
  }
  const bool live = m != -INFINITY;
  const double sstar = __shfl_sync(0xffffffffu, im < 32 ? sv[0] : sv[1], im & 31);
  const double corr = live ? sstar * dot : 0.0;
  const double e2 = 7.38905609893065;  // e^2 (torch's math.exp(2.0))
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = lane + 32 * q;
    if (j < d) {
      double hv = e2 * gv[q];
      if (j == im) hv = hv + (-corr);
      h[o + j] = hv;
      z[o + j] = zv[q];
    }
  }
}

// The adjoint scan's inputs in _chunked_scan's panel layout (inverse of the export): from
// real h (H, S, T, d) float64, out[i][h][r][s nC + cc] = GOOM of h at time t_src, log part
// + (K[h, s] - c[h, s, t_src]) when K is given, with scan time cc L + i and t_src = T - 1 -
// (cc L + i) when reversed. Reads whole d-vectors per state, writes 32-column row segments.
__global__ void __launch_bounds__(256)
    ssm_panels_kernel(const double* __restrict__ hsrc, const double* __restrict__ K,
                      const double* __restrict__ cs, int64_t H, int64_t L, int d, int64_t S,
                      int64_t nC, int64_t T, int reverse, double2* __restrict__ out,
                      int64_t ih0) {
  __shared__ double2 tile[64][kExportCols + 1];
  const int64_t ih = ih0 + blockIdx.y, i = ih / H, h = ih % H, N = S * nC;
  const int64_t n0 = (int64_t)blockIdx.x * kExportCols;
  const int ncols = (int)(N - n0 < kExportCols ? N - n0 : kExportCols);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int j = w; j < ncols; j += 8) {
    const int64_t n = n0 + j, s = n / nC, tin = (n % nC) * L + i;
    const int64_t t = reverse ? T - 1 - tin : tin;
    const int64_t row = (h * S + s) * T + t;
    const double shift = K ? sub_rn(K[h * S + s], cs[row]) : 0.0;
    for (int r = lane; r < d; r += 32) {
      const double v = hsrc[row * d + r];
      double2 g = v == 0.0 ? make_double2(-INFINITY, 0.0)
                           : make_double2(glog(fabs(v)), v < 0.0 ? pi_of<double>() : 0.0);
      if (K) g.x = add_rn(g.x, shift);
      tile[r][j] = g;
    }
  }
  __syncthreads();
  double2* ob = out + ih * d * N + n0;
  for (int e = threadIdx.x; e < d * kExportCols; e += 256) {
    const int r = e / kExportCols, j = e % kExportCols;
    if (j < ncols) ob[(int64_t)r * N + j] = tile[r][j];
  }
}

template <class R>
__global__ void gadd_kernel(const Cx<R>* __restrict__ a, const Cx<R>* __restrict__ b,
                            Cx<R>* __restrict__ out, int64_t n) {
  GRID_STRIDE(i, n) { out[i] = gadd_elem_t<R>(a[i], b[i]); }
}

// one thread per (batch, column); rows looped (columns are contiguous across threads)
template <class R>
__global__ void col_log_norms_kernel(const Cx<R>* __restrict__ z, R* __restrict__ out,
                                     int64_t batch, int rows, int cols) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= batch * cols) return;
  int64_t b = t / cols;
  int c = (int)(t % cols);
  const Cx<R>* zb = z + b * (int64_t)rows * cols + c;
  R top = R(-INFINITY);
  for (int r = 0; r < rows; ++r) top = gmax(top, zb[(int64_t)r * cols].x);
  bool live = top != R(-INFINITY);
  R shift = live ? top : R(0);
  R acc = R(0);
  for (int r = 0; r < rows; ++r) acc += gexp(R(2) * (zb[(int64_t)r * cols].x - shift));
  out[t] = live ? add_rn(shift, R(0.5) * glog(acc)) : R(-INFINITY);
}

// ---- LMME scale pre-pass ---------------------------------------------------
// rows: one warp per (batch, row) -> max(max_j Re A[i, j], 0)
// canonical phase: exactly 0 or pi (what every libgoom kernel emits)
template <class R>
__device__ __forceinline__ bool canonical_phase(R y) {
  return y == R(0) || y == pi_of<R>();
}

template <class R>
__global__ void row_scale_kernel(OperandT<Cx<R>> A, R* __restrict__ out, int64_t batch, int n,
                                 int k, int* __restrict__ noncanon) {
  const int warps = blockDim.x >> 5;
  int64_t w = blockIdx.x * (int64_t)warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= batch * n) return;
  int64_t b = w / n;
  int i = (int)(w % n);
  const Cx<R>* row = A.at(b) + (int64_t)i * k;
  R m = R(-INFINITY);
  bool odd = false;
  for (int j = lane; j < k; j += 32) {
    const Cx<R> z = row[j];
    m = gmax(m, z.x);
    odd |= !canonical_phase(z.y);
  }
  m = warp_max_t(m);
  if (lane == 0) out[w] = gmax(m, R(0));
  if (noncanon && __any_sync(0xffffffffu, odd) && lane == 0) atomicOr(noncanon, 1);
}

// columns: one thread per (batch, column) -> max(max_j Re B[j, c], 0)
template <class R>
__global__ void col_scale_kernel(OperandT<Cx<R>> B, R* __restrict__ out, int64_t batch, int k,
                                 int m, int* __restrict__ noncanon) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool odd = false;
  if (t < batch * m) {
    int64_t b = t / m;
    int c = (int)(t % m);
    const Cx<R>* col = B.at(b) + c;
    R v = R(-INFINITY);
    for (int j = 0; j < k; ++j) {
      const Cx<R> z = col[(int64_t)j * m];
      v = gmax(v, z.x);
      odd |= !canonical_phase(z.y);
    }
    out[t] = gmax(v, R(0));
  }
  if (noncanon && __any_sync(0xffffffffu, odd) && (threadIdx.x & 31) == 0) atomicOr(noncanon, 1);
}

template <class R>
__global__ void identity_kernel(Cx<R>* __restrict__ out, int64_t batch, int d, int64_t stride) {
  const int64_t mat = (int64_t)d * d;
  GRID_STRIDE(i, batch * mat) {
    int64_t b = i / mat, e = i % mat;
    int r = (int)(e / d), c = (int)(e % d);
    out[b * stride + e] = cx<R>(r == c ? R(0) : R(-INFINITY), R(0));
  }
}

__global__ void flags_or_scan_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                     int64_t T) {
  // single CTA: chunked OR-scan (T scan elements; negligible next to the matrix work)
  __shared__ int carry;
  __shared__ int warp_any[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < T; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    int v = (i < T && in) ? (in[i] != 0) : 0;
    unsigned ballot = __ballot_sync(0xffffffffu, v);
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int mine = (ballot & ((2u << lane) - 1u)) != 0;
    if (lane == 31) warp_any[wid] = ballot != 0;
    __syncthreads();
    int before = carry;
    for (int w = 0; w < wid; ++w) before |= warp_any[w];
    if (i < T) out[i] = (uint8_t)(mine | before);
    __syncthreads();
    if (threadIdx.x == 0) {
      int any = carry;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) any |= warp_any[w];
      carry = any;
    }
    __syncthreads();
  }
}

}  // namespace

// ---- host launchers --------------------------------------------------------
template <class R>
int launch_row_scales(OperandT<Cx<R>> A, R* out, int64_t batch, int n, int k, cudaStream_t s,
                      int* noncanon) {
  int64_t warps = batch * n;
  int per_block = 8;
  row_scale_kernel<R><<<(unsigned)((warps + per_block - 1) / per_block), per_block * 32, 0, s>>>(
      A, out, batch, n, k, noncanon);
  GOOM_CHECK_LAUNCH("row_scale_kernel");
  return GOOM_OK;
}

template <class R>
int launch_col_scales(OperandT<Cx<R>> B, R* out, int64_t batch, int k, int m, cudaStream_t s,
                      int* noncanon) {
  int64_t t = batch * m;
  col_scale_kernel<R><<<(unsigned)((t + 255) / 256), 256, 0, s>>>(B, out, batch, k, m, noncanon);
  GOOM_CHECK_LAUNCH("col_scale_kernel");
  return GOOM_OK;
}

template <class R>
int launch_identity(Cx<R>* out, int64_t batch, int d, int64_t stride, cudaStream_t s) {
  identity_kernel<R><<<stream_grid(batch * d * d), kThreads, 0, s>>>(out, batch, d, stride);
  GOOM_CHECK_LAUNCH("identity_kernel");
  return GOOM_OK;
}

template int launch_row_scales<float>(OperandT<float2>, float*, int64_t, int, int, cudaStream_t,
                                      int*);
template int launch_row_scales<double>(OperandT<double2>, double*, int64_t, int, int,
                                       cudaStream_t, int*);
template int launch_col_scales<float>(OperandT<float2>, float*, int64_t, int, int, cudaStream_t,
                                      int*);
template int launch_col_scales<double>(OperandT<double2>, double*, int64_t, int, int,
                                       cudaStream_t, int*);
template int launch_identity<float>(float2*, int64_t, int, int64_t, cudaStream_t);
template int launch_identity<double>(double2*, int64_t, int, int64_t, cudaStream_t);

int launch_flags_or_scan(const uint8_t* in, uint8_t* out, int64_t T, cudaStream_t s) {
  flags_or_scan_kernel<<<1, 1024, 0, s>>>(in, out, T);
  GOOM_CHECK_LAUNCH("flags_or_scan_kernel");
  return GOOM_OK;
}

namespace {

template <class X, class R>
int from_real(const X* x, void* out, int64_t n, X zero_log, void* stream) {
  if (n < 0) return fail(GOOM_EINVAL, "n must be >= 0");
  if (n == 0) return GOOM_OK;
  if (!x || !out) return fail(GOOM_EINVAL, "null pointer");
  from_real_kernel<X, R><<<stream_grid(n), kThreads, 0, as_stream(stream)>>>(
      x, reinterpret_cast<Cx<R>*>(out), n, zero_log);
  GOOM_CHECK_LAUNCH("from_real");
  return GOOM_OK;
}

template <class R, class X>
int to_real(const void* z, X* out, int64_t n, void* stream) {
  if (n < 0) return fail(GOOM_EINVAL, "n must be >= 0");
  if (n == 0) return GOOM_OK;
  if (!z || !out) return fail(GOOM_EINVAL, "null pointer");
  to_real_kernel<R, X><<<stream_grid(n), kThreads, 0, as_stream(stream)>>>(
      reinterpret_cast<const Cx<R>*>(z), out, n);
  GOOM_CHECK_LAUNCH("to_real");
  return GOOM_OK;
}

template <class R>
int to_real_scaled(const void* z, R* out, R* c, int64_t batch, int64_t n, void* stream) {
  if (batch < 0 || n < 0) return fail(GOOM_EINVAL, "batch and n must be >= 0");
  if (batch == 0) return GOOM_OK;
  if (!z || !out || !c) return fail(GOOM_EINVAL, "null pointer");
  to_real_scaled_kernel<R><<<(unsigned)batch, 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const Cx<R>*>(z), out, c, n);
  GOOM_CHECK_LAUNCH("to_real_scaled");
  return GOOM_OK;
}

int ssm_export(const void* X, int64_t H, int64_t L, int d, int64_t S, int64_t nC, int64_t T,
               double* sl, double* ss, double* c, double* z, int reverse, const double* kshift,
               void* stream) {
  if (H < 0 || L < 1 || d < 1 || d > 64 || S < 0 || nC < 0 || T < 0 || T > nC * L)
    return fail(GOOM_ESHAPE, "ssm_export: need 1 <= d <= 64, L >= 1, T <= nC * L");
  if (H == 0 || S == 0 || T == 0) return GOOM_OK;
  if (!X || !sl || !ss) return fail(GOOM_EINVAL, "null pointer");
  // H * L (head, step) rows ride in grid.y, launched in slices of at most 65535
  for (int64_t hi0 = 0; hi0 < H * L; hi0 += 65535) {
    const int64_t rows = H * L - hi0 < 65535 ? H * L - hi0 : 65535;
    const dim3 grid((unsigned)((S * nC + kExportCols - 1) / kExportCols), (unsigned)rows);
    ssm_export_kernel<<<grid, 256, 0, as_stream(stream)>>>(reinterpret_cast<const double2*>(X), L,
                                                          d, S, nC, T, sl, ss, c, z, reverse,
                                                          kshift, hi0);
    GOOM_CHECK_LAUNCH("ssm_export");
  }
  return GOOM_OK;
}

int ssm_panels(const double* h, const double* K, const double* c, int64_t H, int64_t L, int d,
               int64_t S, int64_t nC, int64_t T, int reverse, void* out, void* stream) {
  if (H < 0 || L < 1 || d < 1 || d > 64 || S < 0 || nC < 0 || T != nC * L)
    return fail(GOOM_ESHAPE, "ssm_panels: need 1 <= d <= 64, L >= 1, T == nC * L");
  if (H == 0 || S == 0 || T == 0) return GOOM_OK;
  if (!h || !out || (K && !c)) return fail(GOOM_EINVAL, "null pointer");
  for (int64_t ih0 = 0; ih0 < H * L; ih0 += 65535) {  // grid.y slices of at most 65535
    const int64_t rows = H * L - ih0 < 65535 ? H * L - ih0 : 65535;
    const dim3 grid((unsigned)((S * nC + kExportCols - 1) / kExportCols), (unsigned)rows);
    ssm_panels_kernel<<<grid, 256, 0, as_stream(stream)>>>(h, K, c, H, L, d, S, nC, T, reverse,
                                                          reinterpret_cast<double2*>(out), ih0);
    GOOM_CHECK_LAUNCH("ssm_panels");
  }
  return GOOM_OK;
}

template <class R>
int gadd(const void* a, const void* b, void* out, int64_t n, void* stream) {
  if (n < 0) return fail(GOOM_EINVAL, "n must be >= 0");
  if (n == 0) return GOOM_OK;
  if (!a || !b || !out) return fail(GOOM_EINVAL, "null pointer");
  gadd_kernel<R><<<stream_grid(n), kThreads, 0, as_stream(stream)>>>(
      reinterpret_cast<const Cx<R>*>(a), reinterpret_cast<const Cx<R>*>(b),
      reinterpret_cast<Cx<R>*>(out), n);
  GOOM_CHECK_LAUNCH("gadd");
  return GOOM_OK;
}

template <class R>
int col_log_norms(const void* z, R* out, int64_t batch, int rows, int cols, void* stream) {
  if (batch < 0 || rows < 1 || cols < 1) return fail(GOOM_EINVAL, "bad shape");
  if (batch == 0) return GOOM_OK;
  int64_t t = batch * cols;
  col_log_norms_kernel<R><<<(unsigned)((t + 255) / 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const Cx<R>*>(z), out, batch, rows, cols);
  GOOM_CHECK_LAUNCH("col_log_norms");
  return GOOM_OK;
}

}  // namespace
}  // namespace goom

using namespace goom;

extern "C" {

int goom_from_real_f32(const float* x, goom_c64* out, int64_t n, float zero_log, void* stream) {
  return from_real<float, float>(x, out, n, zero_log, stream);
}
int goom_from_real_f64(const double* x, goom_c64* out, int64_t n, double zero_log, void* stream) {
  return from_real<double, float>(x, out, n, zero_log, stream);
}
int goom_from_real_c128(const double* x, goom_c128* out, int64_t n, double zero_log,
                        void* stream) {
  return from_real<double, double>(x, out, n, zero_log, stream);
}
int goom_to_real_f32(const goom_c64* z, float* out, int64_t n, void* stream) {
  return to_real<float, float>(z, out, n, stream);
}
int goom_to_real_f64(const goom_c64* z, double* out, int64_t n, void* stream) {
  return to_real<float, double>(z, out, n, stream);
}
int goom_to_real_c128(const goom_c128* z, double* out, int64_t n, void* stream) {
  return to_real<double, double>(z, out, n, stream);
}
int goom_to_real_scaled_f32(const goom_c64* z, float* out, float* c, int64_t batch, int64_t n,
                            void* stream) {
  return to_real_scaled<float>(z, out, c, batch, n, stream);
}
int goom_to_real_scaled_c128(const goom_c128* z, double* out, double* c, int64_t batch, int64_t n,
                             void* stream) {
  return to_real_scaled<double>(z, out, c, batch, n, stream);
}
int goom_ssm_export_c128(const goom_c128* X, int64_t H, int64_t L, int d, int64_t S, int64_t nC,
                         int64_t T, double* sl, double* ss, double* c, double* z, int reverse,
                         const double* kshift, void* stream) {
  return ssm_export(X, H, L, d, S, nC, T, sl, ss, c, z, reverse, kshift, stream);
}
int goom_ssm_panels_c128(const double* h, const double* K, const double* c, int64_t H, int64_t L,
                         int d, int64_t S, int64_t nC, int64_t T, int reverse, goom_c128* out,
                         void* stream) {
  return ssm_panels(h, K, c, H, L, d, S, nC, T, reverse, out, stream);
}
int goom_ssm_adjoint_source_f64(const double* sl, const double* ss, const double* c,
                                const double* gz, int64_t n, int d, double* h, double* z,
                                void* stream) {
  if (n < 0 || d < 1 || d > 64) return fail(GOOM_ESHAPE, "ssm_adjoint_source: need 1 <= d <= 64");
  if (n == 0) return GOOM_OK;
  if (!sl || !ss || !c || !gz || !h || !z) return fail(GOOM_EINVAL, "null pointer");
  const int64_t blocks = (n + 7) / 8;  // 8 warps (states) per block
  ssm_adjoint_source_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(sl, ss, c, gz, n, d,
                                                                            h, z);
  GOOM_CHECK_LAUNCH("ssm_adjoint_source");
  return GOOM_OK;
}
int goom_gadd_c64(const goom_c64* a, const goom_c64* b, goom_c64* out, int64_t n, void* stream) {
  return gadd<float>(a, b, out, n, stream);
}
int goom_gadd_c128(const goom_c128* a, const goom_c128* b, goom_c128* out, int64_t n,
                   void* stream) {
  return gadd<double>(a, b, out, n, stream);
}
int goom_col_log_norms_c64(const goom_c64* z, float* out, int64_t batch, int rows, int cols,
                           void* stream) {
  return col_log_norms<float>(z, out, batch, rows, cols, stream);
}
int goom_col_log_norms_c128(const goom_c128* z, double* out, int64_t batch, int rows, int cols,
                            void* stream) {
  return col_log_norms<double>(z, out, batch, rows, cols, stream);
}

}  // extern "C"
