// Internal (non-ABI) interfaces shared across libgoom translation units.
// Everything on the LMME path is generic over the backing precision R
// (float: complex64 GOOMs; double: complex128 GOOMs, the reference's float64).
#pragma once

#include "goom_common.cuh"

namespace goom {

// Signed log-sum-exp of two GOOMs, restating _gadd_arrays (core.py:264-275).
// Explicit _rn intrinsics: no FMA contraction, so the result is bitwise
// commutative (pinned by pkg/tests/test_core.py:327-338).
template <class R>
__device__ __forceinline__ Cx<R> gadd_elem_t(Cx<R> a, Cx<R> b) {
  R top = gmax(a.x, b.x);
  bool live = top != R(-INFINITY);
  R shift = live ? top : R(0);
  // the operand at the top contributes exp(top - top) == 1 exactly (one exp per element,
  // bitwise the same as two); a +inf top keeps exp(inf - inf) = NaN as the two-exp form
  const bool a_top = a.x == top;
  const R e = gexp(sub_rn(a_top ? b.x : a.x, shift));
  const R e_top = top == R(INFINITY) ? R(NAN) : R(1);
  R ea = a_top ? e_top : e;
  R eb = a_top ? e : e_top;
  R t = add_rn(mul_rn(goom_sign_t<R>(a.y), ea), mul_rn(goom_sign_t<R>(b.y), eb));
  if (!live) return cx<R>(R(-INFINITY), R(0));
  return cx<R>(add_rn(shift, glog(fabs(t))), t < R(0) ? pi_of<R>() : R(0));
}
__device__ __forceinline__ float2 gadd_elem(float2 a, float2 b) { return gadd_elem_t<float>(a, b); }

// LMME epilogue: (log|I| + a) + b in this order, as numpy evaluates core.py:259
template <class R>
__device__ __forceinline__ Cx<R> lmme_out(R acc, R a, R b) {
  return cx<R>(add_rn(add_rn(glog(fabs(acc)), a), b), acc < R(0) ? pi_of<R>() : R(0));
}

// Precomputed clamped scales: row scale of the left operand, column scale of the
// right operand, addressed like the operand they belong to (base + (b/div)*stride).
template <class R>
struct ScalesT {
  const R* ptr;
  int64_t stride;
  int64_t div;
  __host__ __device__ __forceinline__ const R* at(int64_t b) const {
    return ptr + (b / div) * stride;
  }
};
using Scales = ScalesT<float>;

template <class R>
struct LmmeProblemT {
  OperandT<Cx<R>> A, B, D;  // D.ptr may be null (no fused gadd)
  Cx<R>* C;
  int64_t strideC;
  int64_t batch;
  int n, k, m;
  ScalesT<R> rowA, colB;    // ptr null -> computed by the pre-pass into workspace
  const int* noncanon;      // device flag from the pre-pass (null: phases unknown)
  // optional (tcgen05 path): clamped row maxima of C into emitRow[b*emitRowStride + i] and
  // column maxima into emitCol[b*emitColStride + j] (atomicMax on the bits; the caller
  // zero-fills), i.e. the scales the next LMME needs when C is its left / right operand
  R* emitRow;
  int64_t emitRowStride;
  R* emitCol;
  int64_t emitColStride;
  // public entry points only: n = m = k = 64 may take the two-products-per-tile tcgen05
  // kernel; the scan / selective engines keep lmme_whole's arithmetic (their bitwise
  // invariants against the CTA-resident engines)
  bool allow_duo;
};
using LmmeProblem = LmmeProblemT<float>;

// ---- tile-scaled fp32 matrices (lmme_ts.cu) ----------------------------------
// The chain engine's internal format: X_ij = U_ij * exp(q[i][j / 256]) with U fp32
// (|U| <= 1 per (row, 256-column block) when produced by an LMME epilogue) and
// G[J] = max_i q[i][J] kept as order-preserving uint bits (float_to_ordered; 0 = unset).
// An LMME of two such matrices needs no exp/log per element: the left operand is
// rescaled per (row, block) by exp(q - rowmax q), the right one per row by exp(q - G),
// and the product's natural scales are rowmax q (left) + G (right).
struct TsIn {
  const float* U;
  const float* q;
  const uint32_t* G;
  int64_t sU, sq, sG;  // per-matrix strides in elements (0 broadcasts one matrix)
  int64_t div;         // matrix index = b / div
};
struct TsOut {
  float* U;
  float* q;
  uint32_t* G;  // caller zero-fills
  int64_t sU, sq, sG;
};
// LMME epilogue targets of the tile-scaled kernel
enum TsOutKind { kTsOutGoom = 0, kTsOutTs = 1, kTsOutDigest = 2 };
struct TsProblem {
  TsIn A, B;
  int kind;
  float2* C;          // kTsOutGoom: complex64 (batch, n, m)
  int64_t strideC;
  TsOut T;            // kTsOutTs
  float4* parts;      // kTsOutDigest: [batch][n / 32][m / 256] (max log, lfro top, sum, bad)
  int64_t batch;
  int n, k, m;
  // chained phase 1 (kTsOutTs only): chain_s > 0 runs L[b s + i] = A[b s + i] (x) L[b s + i - 1]
  // for i = 1 .. chain_s - 1 and every block b < batch in ONE persistent launch; A, B = T = L
  // index chain_T matrices with a one-matrix stride; chain_done: batch x (m / 256) counters,
  // zeroed, completed (row block, CTA) tiles per (block, column tile)
  int chain_s = 0;
  int64_t chain_T = 0;
  uint32_t* chain_done = nullptr;
};
bool lmme_ts_eligible(int n, int k, int m);
// bench instrumentation (chain_ts.cu): CUDA events around a phase of the chain engine,
// recorded only while goom_chain_ts_phase3_timing(1) is on
constexpr int kPhases = 4;
struct PhaseTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t st;
  int ph;
  int64_t n;
  PhaseTimer(cudaStream_t s, int phase, int64_t units);
  void stop();
};
int lmme_ts(const TsProblem& p, cudaStream_t s);
// complex64 GOOM <-> tile-scaled (elementwise, one warp per (row, 256-column block))
int launch_goom_to_ts(const float2* X, int64_t strideX, TsOut out, int64_t batch, int rows,
                      int cols, cudaStream_t s);
int launch_ts_to_goom(TsIn in, float2* X, int64_t strideX, int64_t batch, int rows, int cols,
                      cudaStream_t s);
// the public chain scan on the tile-scaled engine (chain_ts.cu), d % 256 == 0
size_t chain_c64_ts_workspace_bytes(int64_t T, int d, int block);
int chain_scan_c64_ts(const float2* A, float2* out, int64_t T, int d, int block,
                      const float2* carry_in, void* ws, size_t ws_bytes, cudaStream_t st);
// digest partials [batch][parts] -> float4 (max log, log ||.||_F, finite, 0) per matrix
int launch_digest_reduce(const float4* parts, int parts_per, float4* out, int64_t batch,
                         cudaStream_t s);

// ---- launchers (elementwise.cu) ---------------------------------------------
// noncanon (nullable): set to 1 if any imaginary part is not exactly 0 or pi
template <class R>
int launch_row_scales(OperandT<Cx<R>> A, R* out, int64_t batch, int n, int k, cudaStream_t s,
                      int* noncanon = nullptr);
template <class R>
int launch_col_scales(OperandT<Cx<R>> B, R* out, int64_t batch, int k, int m, cudaStream_t s,
                      int* noncanon = nullptr);
// identity matrices at out + b*stride (elements), b < batch
template <class R>
int launch_identity(Cx<R>* out, int64_t batch, int d, int64_t stride, cudaStream_t s);
int launch_flags_or_scan(const uint8_t* in, uint8_t* out, int64_t T, cudaStream_t s);

// ---- LMME (lmme.cu) ---------------------------------------------------------
template <class R>
size_t lmme_workspace_bytes(int64_t batch, int n, int k, int m, int64_t strideA, int64_t divA,
                            int64_t strideB, int64_t divB);
template <class R>
int lmme_run(LmmeProblemT<R> p, void* ws, size_t ws_bytes, cudaStream_t s);
int lmme_backend();

// SIMT kernels (lmme_simt.cu)
template <class R> int lmme_simt_small(const LmmeProblemT<R>& p, cudaStream_t s);
template <class R> int lmme_simt_tiled(const LmmeProblemT<R>& p, cudaStream_t s);
// n, k, m <= 64: one CTA per product, row / column scales fused (no pre-pass)
template <class R> int lmme_simt_whole(const LmmeProblemT<R>& p, cudaStream_t s);
// tcgen05 3xTF32 (lmme_tc.cu), complex64 only; GOOM_EUNSUPPORTED if not tileable
int lmme_tc(const LmmeProblem& p, cudaStream_t s);
bool lmme_tc_eligible(int n, int k, int m);
// one-SM kernel with the scales reduced in-kernel (scale pass through its ring)
bool lmme_tc1_fuse_scales(int n, int k, int m);
// n = m = 64: two products per tcgen05 tile, scales in-kernel (GOOM_EUNSUPPORTED otherwise)
int lmme_tc_duo(const LmmeProblem& p, cudaStream_t s);
// tile-resident long-chain fold for complex64 d = 16 / 32 / 64 on tcgen05 (scan_long_tc.cu):
// chains of s leaves, chain k from carry0 (k = 0) / carries[k - 1], or its first leaf; out:
// every prefix, tot: every chain's last state
bool fold_tc_eligible(int d);
int launch_fold_tc(const float2* A, int64_t T, int d, int64_t s, const float2* carry0,
                   const float2* carries, float2* out, float2* tot, cudaStream_t st);
// cta_group::2 pair-tile variant (lmme_tc2.cu) for n, m multiples of 256; lmme_tc() prefers
// it (GOOM_TC2=0 disables); GOOM_EUNSUPPORTED if the shape / alignment does not fit
int lmme_tc2(const LmmeProblem& p, cudaStream_t s);
bool lmme_tc2_eligible(int n, int k, int m);
// the pair kernel reduces Eq. 11's scales itself (no pre-pass) for this shape
bool lmme_tc2_fuse_scales(int n, int k, int m);

// ---- scans (scan.cu) --------------------------------------------------------
template <class R>
size_t chain_workspace_bytes(int64_t T, int d, int block);
template <class R>
int chain_scan(const Cx<R>* A, Cx<R>* out, int64_t T, int d, int block, const Cx<R>* carry_in,
               void* ws, size_t ws_bytes, cudaStream_t st);
// d <= 32 warp-resident variant (scan_small.cu): L = local products (T), Cx_ = carries (nb+1)
template <class R>
int chain_scan_small(const Cx<R>* A, Cx<R>* out, int64_t T, int d, int64_t s,
                     const Cx<R>* carry_in, Cx<R>* L, Cx<R>* Cx_, cudaStream_t st);
// 32 < d <= 64 CTA-resident variant (scan_cta.cu), same tree and bitwise the same products
bool chain_cta_eligible(int d);
template <class R>
int chain_scan_cta(const Cx<R>* A, Cx<R>* out, int64_t T, int d, int64_t s,
                   const Cx<R>* carry_in, Cx<R>* L, Cx<R>* Cx_, cudaStream_t st);

// d <= 32 (and d = 64 complex64) long-chain engine (scan_long.cu): reduce-then-scan, a
// different fixed tree
template <class R>
bool chain_long_eligible(int d);
template <class R>
size_t chain_long_workspace_bytes(int64_t T, int d);
template <class R>
int chain_scan_long(const Cx<R>* A, Cx<R>* out, int64_t T, int d, const Cx<R>* carry_in,
                    void* ws, size_t ws_bytes, cudaStream_t st);

}  // namespace goom
