// Warp-resident chain scan for small matrices (d <= 32), complex64 and complex128.
//
// One warp owns one block of the reference's two-level tree (_scan_affine_stack,
// scan.py:181-214). Lane l keeps column l of the running prefix in registers, so the
// right operand of every combine never leaves the register file: its column scale is a
// per-lane max, its transformed values are per-lane exps; only the incoming leaf (the
// left operand) is staged through shared memory (row i broadcast to all lanes).
//   k_local  : L[k*s + i] = A[k*s + i] (x) L[k*s + i - 1], sequential per block, blocks in
//              parallel (one warp each)
//   k_carry  : Cx[k+1] = L[last of block k] (x) Cx[k], one warp, sequential over blocks
//   k_apply  : out[t] = L[t] (x) Cx[t / s], a warp per block; the carry is transformed
//              once per block and kept in registers
// Three launches for the whole scan instead of (s - 1) + blocks + 1. Every product uses
// the arithmetic of lmme_small_kernel (per-output FMA chain in ascending k, same
// epilogue), so results are bitwise identical to the generic path.
#include "goom_internal.cuh"

namespace goom {

namespace {

constexpr int kWarps = 4;
constexpr int kPitch = 33;

// Right operand (d x d, column `lane` in registers: log x[i][lane], sign) -> transformed
// column tB[i] = sign * exp(log - b_lane) and the clamped column scale b_lane.
template <class R, int D>
__device__ __forceinline__ R transform_column(const R (&lg)[D], const R (&sg)[D], int d,
                                              R (&tb)[D]) {
  R b = R(-INFINITY);
#pragma unroll
  for (int i = 0; i < D; ++i)
    if (i < d) b = gmax(b, lg[i]);
  b = gmax(b, R(0));
#pragma unroll
  for (int i = 0; i < D; ++i) tb[i] = i < d ? sg[i] * gexp(lg[i] - b) : R(0);
  return b;
}

// C = A (x) B with A (global, d x d) staged via shared memory, B given as the transformed
// column tb / scale bj of lane; result column `lane` into (lg, sg) registers.
template <class R, int D>
__device__ __forceinline__ void warp_lmme(const Cx<R>* __restrict__ a, int d, R* tA, int lane,
                                          const R (&tb)[D], R bj, R (&lg)[D], R (&sg)[D]) {
  // all d row loads in flight at once, then the row reductions (one latency, not d)
  Cx<R> z[D];
#pragma unroll
  for (int i = 0; i < D; ++i)
    z[i] = (i < d && lane < d) ? a[i * d + lane] : cx<R>(R(-INFINITY), R(0));
  R my_ai = R(0);
#pragma unroll
  for (int i = 0; i < D; ++i) {
    if (i < d) {
      R ai = gmax(warp_max_t(z[i].x), R(0));
      if (lane == i) my_ai = ai;
      tA[i * kPitch + lane] = lane < d ? goom_sign_t<R>(z[i].y) * gexp(z[i].x - ai) : R(0);
    }
  }
  __syncwarp();
  R acc[D];
#pragma unroll
  for (int i = 0; i < D; ++i) acc[i] = R(0);
#pragma unroll
  for (int kk = 0; kk < D; ++kk) {
    if (kk < d) {
      const R bv = tb[kk];
#pragma unroll
      for (int i = 0; i < D; ++i)
        if (i < d) acc[i] = gfma(tA[i * kPitch + kk], bv, acc[i]);
    }
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < D; ++i) {
    R ai = __shfl_sync(0xffffffffu, my_ai, i);
    if (i < d) {
      Cx<R> r = lmme_out<R>(acc[i], ai, bj);
      lg[i] = r.x;
      sg[i] = goom_sign_t<R>(r.y);
    }
  }
}

template <class R, int D>
__device__ __forceinline__ void load_column(const Cx<R>* __restrict__ m, int d, int lane,
                                            R (&lg)[D], R (&sg)[D]) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
    if (i < d && lane < d) {
      Cx<R> z = m[i * d + lane];
      lg[i] = z.x;
      sg[i] = goom_sign_t<R>(z.y);
    } else {
      lg[i] = R(-INFINITY);
      sg[i] = R(1);
    }
  }
}

template <class R, int D>
__device__ __forceinline__ void store_column(Cx<R>* __restrict__ m, int d, int lane,
                                             const R (&lg)[D], const R (&sg)[D]) {
  if (lane >= d) return;
#pragma unroll
  for (int i = 0; i < D; ++i)
    if (i < d) m[i * d + lane] = cx<R>(lg[i], sg[i] < R(0) ? pi_of<R>() : R(0));
}

template <class R, int D>
__global__ void __launch_bounds__(kWarps * 32)
    k_local(const Cx<R>* __restrict__ A, Cx<R>* __restrict__ L, int64_t T, int d, int64_t s) {
  __shared__ R tA[kWarps][32 * kPitch];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t blk = blockIdx.x * (int64_t)kWarps + w;
  const int64_t t0 = blk * s;
  if (t0 >= T) return;
  const int64_t mat = (int64_t)d * d;
  const int64_t t1 = t0 + s < T ? t0 + s : T;
  R lg[D], sg[D], tb[D];
  load_column(A + t0 * mat, d, lane, lg, sg);
  store_column(L + t0 * mat, d, lane, lg, sg);
  for (int64_t t = t0 + 1; t < t1; ++t) {
    const R bj = transform_column(lg, sg, d, tb);
    warp_lmme(A + t * mat, d, tA[w], lane, tb, bj, lg, sg);
    store_column(L + t * mat, d, lane, lg, sg);
  }
}

template <class R, int D>
__global__ void __launch_bounds__(32)
    k_carry(const Cx<R>* __restrict__ L, Cx<R>* __restrict__ Cx_, const Cx<R>* __restrict__ carry_in,
            int64_t T, int d, int64_t s, int64_t nb) {
  __shared__ R tA[32 * kPitch];
  const int lane = threadIdx.x;
  const int64_t mat = (int64_t)d * d;
  R lg[D], sg[D], tb[D];
  int64_t k0;
  if (carry_in) {  // Cx[0] = carry_in; Cx[k+1] = L[last_k] (x) Cx[k]
    load_column(carry_in, d, lane, lg, sg);
    store_column(Cx_, d, lane, lg, sg);
    k0 = 0;
  } else {  // Cx[1] = L[s-1]
    load_column(L + (s - 1) * mat, d, lane, lg, sg);
    store_column(Cx_ + mat, d, lane, lg, sg);
    k0 = 1;
  }
  for (int64_t k = k0; k + 1 < nb; ++k) {
    const R bj = transform_column(lg, sg, d, tb);
    warp_lmme(L + (k * s + s - 1) * mat, d, tA, lane, tb, bj, lg, sg);
    store_column(Cx_ + (k + 1) * mat, d, lane, lg, sg);
  }
}

template <class R, int D>
__global__ void __launch_bounds__(kWarps * 32)
    k_apply(const Cx<R>* __restrict__ L, const Cx<R>* __restrict__ Cx_, Cx<R>* __restrict__ out,
            int64_t T, int d, int64_t s, int with_carry) {
  __shared__ R tA[kWarps][32 * kPitch];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t blk = blockIdx.x * (int64_t)kWarps + w;
  const int64_t t0 = blk * s;
  if (t0 >= T) return;
  const int64_t mat = (int64_t)d * d;
  const int64_t t1 = t0 + s < T ? t0 + s : T;
  R lg[D], sg[D], tb[D];
  if (blk == 0 && !with_carry) {  // block 0 is final
    for (int64_t t = t0; t < t1; ++t) {
      load_column(L + t * mat, d, lane, lg, sg);
      store_column(out + t * mat, d, lane, lg, sg);
    }
    return;
  }
  load_column(Cx_ + blk * mat, d, lane, lg, sg);
  const R bj = transform_column(lg, sg, d, tb);
  for (int64_t t = t0; t < t1; ++t) {
    warp_lmme(L + t * mat, d, tA[w], lane, tb, bj, lg, sg);
    store_column(out + t * mat, d, lane, lg, sg);
  }
}

template <class R, int D>
int chain_small_d(const Cx<R>* A, Cx<R>* out, int64_t T, int d, int64_t s, const Cx<R>* carry_in,
                  Cx<R>* L, Cx<R>* Cx_, cudaStream_t st) {
  const int64_t nb = (T + s - 1) / s;
  const unsigned grid = (unsigned)((nb + kWarps - 1) / kWarps);
  k_local<R, D><<<grid, kWarps * 32, 0, st>>>(A, L, T, d, s);
  GOOM_CHECK_LAUNCH("k_local");
  k_carry<R, D><<<1, 32, 0, st>>>(L, Cx_, carry_in, T, d, s, nb);
  GOOM_CHECK_LAUNCH("k_carry");
  k_apply<R, D><<<grid, kWarps * 32, 0, st>>>(L, Cx_, out, T, d, s, carry_in ? 1 : 0);
  GOOM_CHECK_LAUNCH("k_apply");
  return GOOM_OK;
}

}  // namespace

// register capacity bucket: the unrolled loops cover exactly 8, 16 or 32 rows
template <class R>
int chain_scan_small(const Cx<R>* A, Cx<R>* out, int64_t T, int d, int64_t s,
                     const Cx<R>* carry_in, Cx<R>* L, Cx<R>* Cx_, cudaStream_t st) {
  if (d <= 8) return chain_small_d<R, 8>(A, out, T, d, s, carry_in, L, Cx_, st);
  if (d <= 16) return chain_small_d<R, 16>(A, out, T, d, s, carry_in, L, Cx_, st);
  return chain_small_d<R, 32>(A, out, T, d, s, carry_in, L, Cx_, st);
}

template int chain_scan_small<float>(const float2*, float2*, int64_t, int, int64_t, const float2*,
                                     float2*, float2*, cudaStream_t);
template int chain_scan_small<double>(const double2*, double2*, int64_t, int, int64_t,
                                      const double2*, double2*, double2*, cudaStream_t);

}  // namespace goom
