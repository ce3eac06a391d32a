// Elementwise GOOM kernels: real<->GOOM maps, scaled export, signed LSE (gadd),
// column log-norms, and the LMME scale pre-pass (row / column maxima).
//
// All are HBM-bound streaming kernels: 8 B (complex64) per element plus the
// real side; grid-stride loops sized to a multiple of the SM count.
#include "goom_common.cuh"
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

__global__ void from_real_f32_kernel(const float* __restrict__ x, float2* __restrict__ out,
                                     int64_t n, float zero_log) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = x[i];
    out[i] = (v == 0.0f) ? make_float2(zero_log, 0.0f) : goom_from_value(v);
  }
}

__global__ void from_real_f64_kernel(const double* __restrict__ x, float2* __restrict__ out,
                                     int64_t n, double zero_log) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = x[i];
    if (v == 0.0) {
      out[i] = make_float2((float)zero_log, 0.0f);
    } else {
      out[i] = make_float2((float)log(fabs(v)), v < 0.0 ? kPi : 0.0f);
    }
  }
}

__global__ void to_real_f32_kernel(const float2* __restrict__ z, float* __restrict__ out,
                                   int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float2 v = z[i];
    out[i] = goom_sign(v.y) * expf(v.x);
  }
}

__global__ void to_real_f64_kernel(const float2* __restrict__ z, double* __restrict__ out,
                                   int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float2 v = z[i];
    out[i] = (double)goom_sign(v.y) * exp((double)v.x);
  }
}

// one CTA per matrix: max log, then the shifted export
__global__ void to_real_scaled_kernel(const float2* __restrict__ z, float* __restrict__ out,
                                      float* __restrict__ cvec, int64_t n) {
  const int64_t b = blockIdx.x;
  const float2* zb = z + b * n;
  float* ob = out + b * n;
  __shared__ float red[32];
  float m = kNegInf;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmaxf(m, zb[i].x);
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : kNegInf;
    v = warp_max(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  float c = red[0];
  if (c == kNegInf || n == 0) c = 0.0f;
  if (threadIdx.x == 0) cvec[b] = c;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    float2 v = zb[i];
    ob[i] = goom_sign(v.y) * expf(__fadd_rn(__fsub_rn(v.x, c), 2.0f));
  }
}

__global__ void gadd_kernel(const float2* __restrict__ a, const float2* __restrict__ b,
                            float2* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = gadd_elem(a[i], b[i]);
  }
}

// one thread per (batch, column); rows looped (columns are contiguous across threads)
__global__ void col_log_norms_kernel(const float2* __restrict__ z, float* __restrict__ out,
                                     int64_t batch, int rows, int cols) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= batch * cols) return;
  int64_t b = t / cols;
  int c = (int)(t % cols);
  const float2* zb = z + b * (int64_t)rows * cols + c;
  float top = kNegInf;
  for (int r = 0; r < rows; ++r) top = fmaxf(top, zb[(int64_t)r * cols].x);
  bool live = top != kNegInf;
  float shift = live ? top : 0.0f;
  float acc = 0.0f;
  for (int r = 0; r < rows; ++r) acc += expf(2.0f * (zb[(int64_t)r * cols].x - shift));
  out[t] = live ? __fadd_rn(shift, 0.5f * logf(acc)) : kNegInf;
}

// ---- LMME scale pre-pass ---------------------------------------------------
// rows: one warp per (batch, row) -> max(max_j Re A[i, j], 0)
__global__ void row_scale_kernel(Operand A, float* __restrict__ out, int64_t batch, int n,
                                 int k) {
  const int warps = blockDim.x >> 5;
  int64_t w = blockIdx.x * (int64_t)warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= batch * n) return;
  int64_t b = w / n;
  int i = (int)(w % n);
  const float2* row = A.at(b) + (int64_t)i * k;
  float m = kNegInf;
  for (int j = lane; j < k; j += 32) m = fmaxf(m, row[j].x);
  m = warp_max(m);
  if (lane == 0) out[w] = fmaxf(m, 0.0f);
}

// columns: one thread per (batch, column) -> max(max_j Re B[j, c], 0)
__global__ void col_scale_kernel(Operand B, float* __restrict__ out, int64_t batch, int k,
                                 int m) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= batch * m) return;
  int64_t b = t / m;
  int c = (int)(t % m);
  const float2* col = B.at(b) + c;
  float v = kNegInf;
  for (int j = 0; j < k; ++j) v = fmaxf(v, col[(int64_t)j * m].x);
  out[t] = fmaxf(v, 0.0f);
}

__global__ void identity_kernel(float2* __restrict__ out, int64_t batch, int d, int64_t stride) {
  const int64_t mat = (int64_t)d * d;
  int64_t n = batch * mat;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = i / mat, e = i % mat;
    int r = (int)(e / d), c = (int)(e % d);
    out[b * stride + e] = make_float2(r == c ? 0.0f : kNegInf, 0.0f);
  }
}

__global__ void flags_or_scan_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                     int64_t T) {
  // single CTA: chunked OR-scan (T is the number of scan elements; tiny vs matrix work)
  __shared__ int carry;
  __shared__ int warp_any[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < T; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    int v = (i < T && in) ? (in[i] != 0) : 0;
    // inclusive OR-scan inside the CTA via ballots
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
int launch_row_scales(Operand A, float* out, int64_t batch, int n, int k, cudaStream_t s) {
  int64_t warps = batch * n;
  int per_block = 8;
  row_scale_kernel<<<(unsigned)((warps + per_block - 1) / per_block), per_block * 32, 0, s>>>(
      A, out, batch, n, k);
  GOOM_CHECK_LAUNCH("row_scale_kernel");
  return GOOM_OK;
}

int launch_col_scales(Operand B, float* out, int64_t batch, int k, int m, cudaStream_t s) {
  int64_t t = batch * m;
  col_scale_kernel<<<(unsigned)((t + 255) / 256), 256, 0, s>>>(B, out, batch, k, m);
  GOOM_CHECK_LAUNCH("col_scale_kernel");
  return GOOM_OK;
}

int launch_identity(float2* out, int64_t batch, int d, int64_t stride, cudaStream_t s) {
  identity_kernel<<<stream_grid(batch * d * d), kThreads, 0, s>>>(out, batch, d, stride);
  GOOM_CHECK_LAUNCH("identity_kernel");
  return GOOM_OK;
}

int launch_flags_or_scan(const uint8_t* in, uint8_t* out, int64_t T, cudaStream_t s) {
  flags_or_scan_kernel<<<1, 1024, 0, s>>>(in, out, T);
  GOOM_CHECK_LAUNCH("flags_or_scan_kernel");
  return GOOM_OK;
}

int launch_gadd(const float2* a, const float2* b, float2* out, int64_t n, cudaStream_t s) {
  if (n == 0) return GOOM_OK;
  gadd_kernel<<<stream_grid(n), kThreads, 0, s>>>(a, b, out, n);
  GOOM_CHECK_LAUNCH("gadd_kernel");
  return GOOM_OK;
}

}  // namespace goom

using namespace goom;

extern "C" {

int goom_from_real_f32(const float* x, goom_c64* out, int64_t n, float zero_log, void* stream) {
  if (n < 0) return fail(GOOM_EINVAL, "n must be >= 0");
  if (n == 0) return GOOM_OK;
  if (!x || !out) return fail(GOOM_EINVAL, "null pointer");
  from_real_f32_kernel<<<stream_grid(n), kThreads, 0, as_stream(stream)>>>(
      x, reinterpret_cast<float2*>(out), n, zero_log);
  GOOM_CHECK_LAUNCH("from_real_f32");
  return GOOM_OK;
}

int goom_from_real_f64(const double* x, goom_c64* out, int64_t n, double zero_log, void* stream) {
  if (n < 0) return fail(GOOM_EINVAL, "n must be >= 0");
  if (n == 0) return GOOM_OK;
  if (!x || !out) return fail(GOOM_EINVAL, "null pointer");
  from_real_f64_kernel<<<stream_grid(n), kThreads, 0, as_stream(stream)>>>(
      x, reinterpret_cast<float2*>(out), n, zero_log);
  GOOM_CHECK_LAUNCH("from_real_f64");
  return GOOM_OK;
}

int goom_to_real_f32(const goom_c64* z, float* out, int64_t n, void* stream) {
  if (n < 0) return fail(GOOM_EINVAL, "n must be >= 0");
  if (n == 0) return GOOM_OK;
  if (!z || !out) return fail(GOOM_EINVAL, "null pointer");
  to_real_f32_kernel<<<stream_grid(n), kThreads, 0, as_stream(stream)>>>(
      reinterpret_cast<const float2*>(z), out, n);
  GOOM_CHECK_LAUNCH("to_real_f32");
  return GOOM_OK;
}

int goom_to_real_f64(const goom_c64* z, double* out, int64_t n, void* stream) {
  if (n < 0) return fail(GOOM_EINVAL, "n must be >= 0");
  if (n == 0) return GOOM_OK;
  if (!z || !out) return fail(GOOM_EINVAL, "null pointer");
  to_real_f64_kernel<<<stream_grid(n), kThreads, 0, as_stream(stream)>>>(
      reinterpret_cast<const float2*>(z), out, n);
  GOOM_CHECK_LAUNCH("to_real_f64");
  return GOOM_OK;
}

int goom_to_real_scaled_f32(const goom_c64* z, float* out, float* c, int64_t batch, int64_t n,
                            void* stream) {
  if (batch < 0 || n < 0) return fail(GOOM_EINVAL, "batch and n must be >= 0");
  if (batch == 0) return GOOM_OK;
  if (!z || !out || !c) return fail(GOOM_EINVAL, "null pointer");
  to_real_scaled_kernel<<<(unsigned)batch, 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float2*>(z), out, c, n);
  GOOM_CHECK_LAUNCH("to_real_scaled");
  return GOOM_OK;
}

int goom_gadd_c64(const goom_c64* a, const goom_c64* b, goom_c64* out, int64_t n, void* stream) {
  if (n < 0) return fail(GOOM_EINVAL, "n must be >= 0");
  if (n && (!a || !b || !out)) return fail(GOOM_EINVAL, "null pointer");
  return launch_gadd(reinterpret_cast<const float2*>(a), reinterpret_cast<const float2*>(b),
                     reinterpret_cast<float2*>(out), n, as_stream(stream));
}

int goom_col_log_norms_c64(const goom_c64* z, float* out, int64_t batch, int rows, int cols,
                           void* stream) {
  if (batch < 0 || rows < 1 || cols < 1) return fail(GOOM_EINVAL, "bad shape");
  if (batch == 0) return GOOM_OK;
  int64_t t = batch * cols;
  col_log_norms_kernel<<<(unsigned)((t + 255) / 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float2*>(z), out, batch, rows, cols);
  GOOM_CHECK_LAUNCH("col_log_norms");
  return GOOM_OK;
}

}  // extern "C"
