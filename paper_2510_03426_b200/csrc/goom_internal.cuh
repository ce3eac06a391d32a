// Internal (non-ABI) interfaces shared across libgoom translation units.
#pragma once

#include "goom_common.cuh"

namespace goom {

// Signed log-sum-exp of two GOOMs, restating _gadd_arrays (core.py:264-275).
// Explicit _rn intrinsics: no FMA contraction, so the result is bitwise
// commutative (pinned by pkg/tests/test_core.py:327-338).
__device__ __forceinline__ float2 gadd_elem(float2 a, float2 b) {
  float top = fmaxf(a.x, b.x);
  bool live = top != kNegInf;
  float shift = live ? top : 0.0f;
  float ea = expf(__fsub_rn(a.x, shift));
  float eb = expf(__fsub_rn(b.x, shift));
  float t = __fadd_rn(__fmul_rn(goom_sign(a.y), ea), __fmul_rn(goom_sign(b.y), eb));
  if (!live) return make_float2(kNegInf, 0.0f);
  return make_float2(__fadd_rn(shift, logf(fabsf(t))), t < 0.0f ? kPi : 0.0f);
}

// ---- launchers (elementwise.cu) ---------------------------------------------
int launch_row_scales(Operand A, float* out, int64_t batch, int n, int k, cudaStream_t s);
int launch_col_scales(Operand B, float* out, int64_t batch, int k, int m, cudaStream_t s);
// identity matrices at out + b*stride (elements), b < batch
int launch_identity(float2* out, int64_t batch, int d, int64_t stride, cudaStream_t s);
int launch_flags_or_scan(const uint8_t* in, uint8_t* out, int64_t T, cudaStream_t s);
int launch_gadd(const float2* a, const float2* b, float2* out, int64_t n, cudaStream_t s);

// ---- LMME (lmme.cu) ---------------------------------------------------------
// Precomputed clamped scales: row scale of the left operand, column scale of the
// right operand, addressed like the operand they belong to (base + (b/div)*stride).
struct Scales {
  const float* ptr;
  int64_t stride;
  int64_t div;
  __host__ __device__ __forceinline__ const float* at(int64_t b) const {
    return ptr + (b / div) * stride;
  }
};

struct LmmeProblem {
  Operand A, B, D;      // D.ptr may be null (no fused gadd)
  float2* C;
  int64_t strideC;
  int64_t batch;
  int n, k, m;
  Scales rowA, colB;    // ptr null -> computed by the pre-pass into workspace
};

size_t lmme_workspace_bytes(int64_t batch, int n, int k, int m, const Operand& A,
                            const Operand& B);
int lmme_run(LmmeProblem p, void* ws, size_t ws_bytes, cudaStream_t s);
int lmme_backend();

// SIMT kernels (lmme_simt.cu)
int lmme_simt_small(const LmmeProblem& p, cudaStream_t s);    // n,k,m <= 32, scales in-kernel
int lmme_simt_tiled(const LmmeProblem& p, cudaStream_t s);    // any shape, scales given
// tcgen05 3xTF32 (lmme_tc.cu); returns GOOM_EUNSUPPORTED if the shape is not tileable
int lmme_tc(const LmmeProblem& p, cudaStream_t s);
bool lmme_tc_eligible(int n, int k, int m);

}  // namespace goom
