// CTA-resident chain scan for 33 <= d <= 64, complex64 and complex128.
//
// The reference's two-level tree (_scan_affine_stack, scan.py:181-214) with the running
// right operand of every sequential walk kept in shared memory instead of HBM:
//   k_walk (phase 1) one CTA per block: L[ks+i] = A[ks+i] (x) L[ks+i-1], i = 1..s-1; the
//                    running product never leaves the CTA (it is the next step's right
//                    operand), only the leaf is read and L written: 16 d^2 B per element
//                    where the batched form reads A, L and writes L (24 d^2 B)
//   k_walk (phase 2) one CTA: Cx[k+1] = L[last of block k] (x) Cx[k], the sequential fold
//   k_apply (phase 3) one CTA per block: out[t] = L[t] (x) Cx[t / s]; the carry's column
//                    scales and exponentials are computed ONCE per block and stay in shared
//                    memory (the batched form re-reads and re-exponentiates it per product)
// Three launches for the whole scan instead of (s - 1) + nb + 1. Every product uses the
// arithmetic of lmme_whole_kernel (lmme_simt.cu): clamped row / column maxima (Eq. 11),
// sign * exp(log - scale) operands, a 4 x 4 register tile per thread with one FMA per term
// in ascending k, the lmme_out epilogue — so the results are bitwise identical to the
// generic path's batched launches (test_gpu_scan.py checks it).
#include "goom_internal.cuh"

namespace goom {

namespace {

constexpr int kP = 68;          // shared-memory pitch (64 + 4, as lmme_whole_kernel)
constexpr int kThreads = 256;   // 16 x 16 threads, 4 x 4 outputs each
constexpr int kPer = 64 * 64 / kThreads;  // leaf elements per thread (d <= 64)

template <class R>
struct Smem {
  R a[64 * kP];            // left operand, [kk][row]: log, then sign * exp(log - a_i)
  R b[64 * kP];            // right operand, [kk][col]: log, then sign * exp(log - b_j)
  R sc[128];               // a_i (0..63), b_j (64..127)
  signed char ga[64 * kP];  // signs of a
  signed char gb[64 * kP];  // signs of b
};

template <class R>
__device__ __forceinline__ void lds4r(const R* p, R (&v)[4]) {
  if constexpr (sizeof(R) == 4) {
    const float4 q = *reinterpret_cast<const float4*>(p);
    v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
  } else {
    const double2 q0 = *reinterpret_cast<const double2*>(p);
    const double2 q1 = *reinterpret_cast<const double2*>(p + 2);
    v[0] = q0.x, v[1] = q0.y, v[2] = q1.x, v[3] = q1.y;
  }
}

// d x d row-major matrix -> registers (coalesced: element tid + 256 r)
template <class R>
__device__ __forceinline__ void fetch(const Cx<R>* __restrict__ x, int dd, Cx<R> (&v)[kPer]) {
#pragma unroll
  for (int r = 0; r < kPer; ++r) {
    const int e = threadIdx.x + kThreads * r;
    v[r] = e < dd ? x[e] : cx<R>(R(-INFINITY), R(0));
  }
}

// registers -> [kk][row] log plane + signs (left operand: row i, column kk of x)
template <class R>
__device__ __forceinline__ void stage_left(const Cx<R> (&v)[kPer], int d, Smem<R>& s) {
#pragma unroll
  for (int r = 0; r < kPer; ++r) {
    const int e = threadIdx.x + kThreads * r;
    if (e < d * d) {
      const int i = e / d, kk = e % d;
      s.a[kk * kP + i] = v[r].x;
      s.ga[kk * kP + i] = goom_sign_t<R>(v[r].y) < R(0) ? -1 : 1;
    }
  }
}

// registers -> [kk][col] log plane + signs (right operand: row kk, column j)
template <class R>
__device__ __forceinline__ void stage_right(const Cx<R> (&v)[kPer], int d, Smem<R>& s) {
#pragma unroll
  for (int r = 0; r < kPer; ++r) {
    const int e = threadIdx.x + kThreads * r;
    if (e < d * d) {
      const int kk = e / d, j = e % d;
      s.b[kk * kP + j] = v[r].x;
      s.gb[kk * kP + j] = goom_sign_t<R>(v[r].y) < R(0) ? -1 : 1;
    }
  }
}

// clamped maxima (Eq. 11, core.py:252-253): rows of a (threads 0..63) and / or columns of
// b (threads 64..127), then the exponentials in place
template <class R>
__device__ __forceinline__ void scales_and_exp(int d, Smem<R>& s, bool do_a, bool do_b) {
  const int tid = threadIdx.x;
  if (do_a && tid < 64) {
    R v = R(-INFINITY);
    if (tid < d)
      for (int kk = 0; kk < d; ++kk) v = gmax(v, s.a[kk * kP + tid]);
    s.sc[tid] = gmax(v, R(0));
  } else if (do_b && tid >= 64 && tid < 128) {
    const int j = tid - 64;
    R v = R(-INFINITY);
    if (j < d)
      for (int kk = 0; kk < d; ++kk) v = gmax(v, s.b[kk * kP + j]);
    s.sc[tid] = gmax(v, R(0));
  }
  __syncthreads();
  for (int e = tid; e < 64 * d; e += kThreads) {
    const int kk = e >> 6, c = e & 63;
    const int o = kk * kP + c;
    if (do_a) s.a[o] = c < d ? R(s.ga[o]) * gexp(s.a[o] - s.sc[c]) : R(0);
    if (do_b) s.b[o] = c < d ? R(s.gb[o]) * gexp(s.b[o] - s.sc[64 + c]) : R(0);
  }
  __syncthreads();
}

// the 4 x 4 tile of this thread (rows 4 ty .., columns 4 tx ..), ascending kk
template <class R>
__device__ __forceinline__ void gemm(int d, const Smem<R>& s, R (&acc)[4][4]) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = R(0);
  for (int kk = 0; kk < d; ++kk) {
    R ar[4], br[4];
    lds4r(&s.a[kk * kP + ty * 4], ar);
    lds4r(&s.b[kk * kP + tx * 4], br);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = gfma(ar[i], br[j], acc[i][j]);
  }
}

// epilogue: out = lmme_out(acc, a_i, b_j) -> global (row-major d x d) and, when `keep`,
// into the right-operand planes as the next step's right operand (its rows are the kk)
template <class R>
__device__ __forceinline__ void finish(int d, Smem<R>& s, const R (&acc)[4][4],
                                       Cx<R>* __restrict__ out, bool keep) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  Cx<R> o[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = ty * 4 + i, c = tx * 4 + j;
      o[i][j] = lmme_out<R>(acc[i][j], s.sc[r < 64 ? r : 0], s.sc[64 + c]);
      if (r < d && c < d) out[(int64_t)r * d + c] = o[i][j];
    }
  if (!keep) return;
  __syncthreads();  // every thread's GEMM reads of b and its scale reads are done
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = ty * 4 + i, c = tx * 4 + j;
      if (r < d && c < d) {
        s.b[r * kP + c] = o[i][j].x;
        s.gb[r * kP + c] = goom_sign_t<R>(o[i][j].y) < R(0) ? -1 : 1;
      }
    }
}

// Walk: chain c (blockIdx.x) has left operands X[c*xs + i*xi] for i = 1 .. n_c - 1 and the
// initial right operand R0 = init (or X[c*xs] itself when init is null); it writes
// R_i = X_i (x) R_{i-1} to Y[c*ys + i*yi] (R_0 not written). n_c = min(n, total - c*n) in
// units of steps of the global sequence of length `total` (the last block may be short).
template <class R>
__global__ void __launch_bounds__(kThreads)
    k_walk(const Cx<R>* __restrict__ X, int64_t xs, int64_t xi, const Cx<R>* __restrict__ init,
           Cx<R>* __restrict__ Y, int64_t ys, int64_t yi, int64_t n, int64_t total, int d) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<R>& s = *reinterpret_cast<Smem<R>*>(smem_raw);
  const int64_t c = blockIdx.x;
  const int64_t steps = (total - c * n < n ? total - c * n : n);
  const int64_t mat = (int64_t)d * d;
  const int dd = d * d;
  const Cx<R>* x = X + c * xs;
  Cx<R> v[kPer];
  fetch<R>(init ? init : x, dd, v);
  stage_right<R>(v, d, s);
  if (steps > 1) fetch<R>(x + xi * mat, dd, v);
  for (int64_t i = 1; i < steps; ++i) {
    stage_left<R>(v, d, s);
    __syncthreads();
    if (i + 1 < steps) fetch<R>(x + (i + 1) * xi * mat, dd, v);  // next leaf in flight
    scales_and_exp<R>(d, s, true, true);
    R acc[4][4];
    gemm<R>(d, s, acc);
    finish<R>(d, s, acc, Y + c * ys + i * yi * mat, true);
    __syncthreads();
  }
}

// Apply: block c of out[t] = L[t] (x) C[c] for t in [c s, min((c+1) s, T)); C[c] at
// C + c * cs (cs = 0: one carry for every block); t < skip are copied from L (block 0
// without a carry-in)
template <class R>
__global__ void __launch_bounds__(kThreads)
    k_apply(const Cx<R>* __restrict__ L, const Cx<R>* __restrict__ C, int64_t cs,
            Cx<R>* __restrict__ out, int64_t s_len, int64_t T, int64_t skip, int d) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<R>& s = *reinterpret_cast<Smem<R>*>(smem_raw);
  const int64_t c = blockIdx.x;
  const int64_t t0 = c * s_len;
  const int64_t t1 = (t0 + s_len < T ? t0 + s_len : T);
  const int64_t mat = (int64_t)d * d;
  const int dd = d * d;
  if (t1 <= skip) {  // a block without a carry: its prefixes are its local products
    for (int64_t e = threadIdx.x; e < (t1 - t0) * mat; e += kThreads) out[t0 * mat + e] = L[t0 * mat + e];
    return;
  }
  Cx<R> v[kPer];
  fetch<R>(C + c * cs, dd, v);
  stage_right<R>(v, d, s);
  __syncthreads();
  scales_and_exp<R>(d, s, false, true);  // the carry's scales and exponentials, once per block
  fetch<R>(L + t0 * mat, dd, v);
  for (int64_t t = t0; t < t1; ++t) {
    stage_left<R>(v, d, s);
    __syncthreads();
    if (t + 1 < t1) fetch<R>(L + (t + 1) * mat, dd, v);
    scales_and_exp<R>(d, s, true, false);
    R acc[4][4];
    gemm<R>(d, s, acc);
    finish<R>(d, s, acc, out + t * mat, false);
    __syncthreads();
  }
}

template <class R>
int smem_setup() {
  GOOM_TRY(smem_attr((const void*)k_walk<R>, (int)sizeof(Smem<R>), "scan_cta smem attribute"));
  GOOM_TRY(smem_attr((const void*)k_apply<R>, (int)sizeof(Smem<R>), "scan_cta smem attribute"));
  return GOOM_OK;
}

template <class C>
int copy_rows(C* dst, const C* src, size_t width, size_t pitch, size_t rows, cudaStream_t st) {
  if (rows && cudaMemcpy2DAsync(dst, sizeof(C) * pitch, src, sizeof(C) * pitch, sizeof(C) * width,
                                rows, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "scan_cta copy");
  return GOOM_OK;
}

}  // namespace

bool chain_cta_eligible(int d) { return d > 32 && d <= 64; }

// A (T, d, d) -> out (T, d, d), block s, optional carry_in (right, applied to every prefix);
// L (T mats) and Cx (nb + 1 mats) are workspace, as chain_scan's
template <class R>
int chain_scan_cta(const Cx<R>* A, Cx<R>* out, int64_t T, int d, int64_t s,
                   const Cx<R>* carry_in, Cx<R>* L, Cx<R>* Cx_, cudaStream_t st) {
  using C = Cx<R>;
  if (!chain_cta_eligible(d)) return fail(GOOM_EUNSUPPORTED, "scan_cta needs 32 < d <= 64");
  GOOM_TRY(smem_setup<R>());
  const int64_t mat = (int64_t)d * d;
  const int64_t nb = (T + s - 1) / s;
  const size_t smem = sizeof(Smem<R>);
  // phase 1: L[ks] = A[ks]; the walk writes L[ks+1 .. ks+s-1]
  GOOM_TRY(copy_rows(L, A, mat, mat * s, nb, st));
  if (s > 1) {
    k_walk<R><<<(unsigned)nb, kThreads, smem, st>>>(A, s * mat, 1, nullptr, L, s * mat, 1, s, T, d);
    GOOM_CHECK_LAUNCH("scan_cta k_walk (phase 1)");
  }
  // phase 2: Cx[1] = L[s-1] (no carry) or L[s-1] (x) carry_in; Cx[k+1] = L[last_k] (x) Cx[k]
  // — one walk over the block ends: left operands L[s-1], L[2s-1], ... (stride s), the last
  // block's end clamped by the walk's own length (its last left operand is L[T-1] only when
  // the last block is full; otherwise Cx[nb] is not needed by phase 3)
  if (carry_in) {
    GOOM_TRY(copy_rows(Cx_, carry_in, mat, mat, 1, st));
    if (nb > 1) {
      // Cx[k+1] = L[ks + s - 1] (x) Cx[k] for k = 0 .. nb - 2: walk with X_i = L[(i-1)s + s-1]
      k_walk<R><<<1, kThreads, smem, st>>>(L + (s - 1) * mat - s * mat, 0, s, carry_in, Cx_, 0, 1,
                                           nb, nb, d);
      GOOM_CHECK_LAUNCH("scan_cta k_walk (phase 2)");
    }
  } else if (nb > 1) {
    GOOM_TRY(copy_rows(Cx_ + mat, L + (s - 1) * mat, mat, mat, 1, st));
    if (nb > 2) {
      // Cx[k+1] = L[ks + s - 1] (x) Cx[k] for k = 1 .. nb - 2: X_i = L[i s + s - 1], R_0 = Cx[1]
      k_walk<R><<<1, kThreads, smem, st>>>(L + (s - 1) * mat, 0, s, Cx_ + mat, Cx_ + mat, 0, 1,
                                           nb - 1, nb - 1, d);
      GOOM_CHECK_LAUNCH("scan_cta k_walk (phase 2)");
    }
  }
  // phase 3: out[t] = L[t] (x) Cx[t / s] (block 0 without a carry: copied)
  k_apply<R><<<(unsigned)nb, kThreads, smem, st>>>(L, Cx_, mat, out, s, T, carry_in ? 0 : s, d);
  GOOM_CHECK_LAUNCH("scan_cta k_apply");
  return GOOM_OK;
}

template int chain_scan_cta<float>(const float2*, float2*, int64_t, int, int64_t, const float2*,
                                   float2*, float2*, cudaStream_t);
template int chain_scan_cta<double>(const double2*, double2*, int64_t, int, int64_t,
                                    const double2*, double2*, double2*, cudaStream_t);

}  // namespace goom
