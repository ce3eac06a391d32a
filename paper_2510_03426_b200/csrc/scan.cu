// Blocked prefix-scan engines over LMME combines.
//
// Both engines use the reference's two-level tree (_scan_affine_stack,
// scan.py:181-214) with block s, restructured for the GPU:
//   phase 1  local inclusive scans inside every block, batched across blocks
//            (s-1 batched LMME launches; one product per block per launch);
//   phase 2  the sequential fold of block carries, touching ONLY the last
//            element of each block (nblocks single-product launches);
//   phase 3  one batched launch applying carry(k-1) to every element of block k.
// Phase 2+3 perform exactly the reference's level-2 combines (each element of
// block k is combined with the final value of element k*s-1), so the combine
// tree — and hence the floating-point structure — matches the reference for
// the same block size. Products accumulate on the left: out[t] = A_t ... A_0.
//
// Buffers: local products L (T matrices) and carries Cx (nblocks+1) live in the
// caller's workspace; the input is never written; out may not alias the input.
#include "goom_internal.cuh"

namespace goom {

namespace {

inline size_t round_up(size_t x) { return (x + 255) & ~size_t(255); }

struct Carve {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    T* p = reinterpret_cast<T*>(base + off);
    off += round_up(sizeof(T) * count);
    return p;
  }
};

size_t lmme_ws(int64_t batch, int n, int k, int m) {
  // worst case: every operand distinct
  return round_up(sizeof(float) * (size_t)batch * n) + round_up(sizeof(float) * (size_t)batch * m);
}

// out[b] = A(b) (x) B(b) (+) D(b)
int lmme_call(Operand A, Operand B, Operand D, float2* C, int64_t strideC, int64_t batch, int n,
              int k, int m, void* ws, size_t ws_bytes, cudaStream_t s) {
  LmmeProblem p{};
  p.A = A;
  p.B = B;
  p.D = D;
  p.C = C;
  p.strideC = strideC;
  p.batch = batch;
  p.n = n;
  p.k = k;
  p.m = m;
  p.rowA = Scales{nullptr, 0, 1};
  p.colB = Scales{nullptr, 0, 1};
  return lmme_run(p, ws, ws_bytes, s);
}

const Operand kNone{nullptr, 0, 1};

}  // namespace

size_t chain_workspace_bytes(int64_t T, int d, int block) {
  int64_t s = block < T ? block : T;
  int64_t nb = (T + s - 1) / s;
  size_t mat = (size_t)d * d;
  size_t lm = lmme_ws(T, d, d, d);
  return round_up(sizeof(float2) * mat * T) + round_up(sizeof(float2) * mat * (nb + 1)) + lm;
}

// Product chain with optional right carry (see header comment).
int chain_scan(const float2* A, float2* out, int64_t T, int d, int block, const float2* carry_in,
               void* ws, size_t ws_bytes, cudaStream_t st) {
  const int64_t s = block < T ? block : T;
  const int64_t nb = (T + s - 1) / s;
  const int64_t mat = (int64_t)d * d;
  if (ws_bytes < chain_workspace_bytes(T, d, block))
    return fail(GOOM_EWORKSPACE, "chain scan workspace too small");
  Carve cv{reinterpret_cast<char*>(ws)};
  float2* L = cv.take<float2>((size_t)mat * T);
  float2* Cx = cv.take<float2>((size_t)mat * (nb + 1));
  void* lws = cv.base + cv.off;
  size_t lws_bytes = ws_bytes - cv.off;

  // phase 1: L[k*s] = A[k*s]; L[k*s+i] = A[k*s+i] (x) L[k*s+i-1]
  if (cudaMemcpy2DAsync(L, sizeof(float2) * mat * s, A, sizeof(float2) * mat * s,
                        sizeof(float2) * mat, nb, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "chain phase-1 copy");
  for (int64_t i = 1; i < s; ++i) {
    int64_t cnt = (T - i + s - 1) / s;  // blocks whose length exceeds i
    if (cnt <= 0) break;
    GOOM_TRY(lmme_call(Operand{A + i * mat, s * mat, 1}, Operand{L + (i - 1) * mat, s * mat, 1},
                       kNone, L + i * mat, s * mat, cnt, d, d, d, lws, lws_bytes, st));
  }
  // phase 2: Cx[0] = carry_in; Cx[k+1] = L[last of block k] (x) Cx[k]
  for (int64_t kb = 0; kb < nb; ++kb) {
    int64_t last = (kb * s + s < T ? kb * s + s : T) - 1;
    if (kb == 0 && !carry_in) {
      if (cudaMemcpyAsync(Cx + mat, L + last * mat, sizeof(float2) * mat,
                          cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return cuda_fail(cudaGetLastError(), "chain carry copy");
      continue;
    }
    const float2* prev = (kb == 0) ? carry_in : Cx + kb * mat;
    if (kb == nb - 1) break;  // the last block's carry-out is produced by phase 3
    GOOM_TRY(lmme_call(Operand{L + last * mat, 0, 1}, Operand{prev, 0, 1}, kNone,
                       Cx + (kb + 1) * mat, 0, 1, d, d, d, lws, lws_bytes, st));
  }
  // phase 3: out[b] = L[b] (x) Cx[b/s]  (block 0 needs a carry only with carry_in)
  if (carry_in) {
    if (cudaMemcpyAsync(Cx, carry_in, sizeof(float2) * mat, cudaMemcpyDeviceToDevice, st) !=
        cudaSuccess)
      return cuda_fail(cudaGetLastError(), "chain carry-in copy");
    GOOM_TRY(lmme_call(Operand{L, mat, 1}, Operand{Cx, mat, s}, kNone, out, mat, T, d, d, d, lws,
                       lws_bytes, st));
  } else {
    if (cudaMemcpyAsync(out, L, sizeof(float2) * mat * s, cudaMemcpyDeviceToDevice, st) !=
        cudaSuccess)
      return cuda_fail(cudaGetLastError(), "chain block-0 copy");
    if (T > s)
      GOOM_TRY(lmme_call(Operand{L + s * mat, mat, 1}, Operand{Cx + mat, mat, s}, kNone,
                         out + s * mat, mat, T - s, d, d, d, lws, lws_bytes, st));
  }
  return GOOM_OK;
}

size_t affine_workspace_bytes(int64_t T, int d, int m, int block) {
  int64_t s = block < T ? block : T;
  int64_t nb = (T + s - 1) / s;
  size_t lm = lmme_ws(T, d, d, d > m ? d : m);
  return round_up(sizeof(float2) * (size_t)d * d * T) + round_up(sizeof(float2) * (size_t)d * m * T) +
         round_up(sizeof(float2) * (size_t)d * d * (nb + 1)) +
         round_up(sizeof(float2) * (size_t)d * m * (nb + 1)) + lm;
}

int affine_scan(const float2* A, const float2* B, const uint8_t* flags_in, float2* outA,
                float2* outB, uint8_t* flags_out, int64_t T, int d, int m, int block, void* ws,
                size_t ws_bytes, cudaStream_t st) {
  const int64_t s = block < T ? block : T;
  const int64_t nb = (T + s - 1) / s;
  const int64_t ma = (int64_t)d * d, mb = (int64_t)d * m;
  if (ws_bytes < affine_workspace_bytes(T, d, m, block))
    return fail(GOOM_EWORKSPACE, "affine scan workspace too small");
  Carve cv{reinterpret_cast<char*>(ws)};
  float2* LA = cv.take<float2>((size_t)ma * T);
  float2* LB = cv.take<float2>((size_t)mb * T);
  float2* CA = cv.take<float2>((size_t)ma * (nb + 1));
  float2* CB = cv.take<float2>((size_t)mb * (nb + 1));
  void* lws = cv.base + cv.off;
  size_t lws_bytes = ws_bytes - cv.off;

  if (cudaMemcpy2DAsync(LA, sizeof(float2) * ma * s, A, sizeof(float2) * ma * s,
                        sizeof(float2) * ma, nb, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
      cudaMemcpy2DAsync(LB, sizeof(float2) * mb * s, B, sizeof(float2) * mb * s,
                        sizeof(float2) * mb, nb, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "affine phase-1 copy");
  // phase 1 (combine_affine, scan.py:173-178): A slot then fused bias slot
  for (int64_t i = 1; i < s; ++i) {
    int64_t cnt = (T - i + s - 1) / s;
    if (cnt <= 0) break;
    Operand cur{A + i * ma, s * ma, 1};
    GOOM_TRY(lmme_call(cur, Operand{LA + (i - 1) * ma, s * ma, 1}, kNone, LA + i * ma, s * ma, cnt,
                       d, d, d, lws, lws_bytes, st));
    GOOM_TRY(lmme_call(cur, Operand{LB + (i - 1) * mb, s * mb, 1}, Operand{B + i * mb, s * mb, 1},
                       LB + i * mb, s * mb, cnt, d, d, m, lws, lws_bytes, st));
  }
  // phase 2: carries
  for (int64_t kb = 0; kb + 1 < nb; ++kb) {
    int64_t last = kb * s + s - 1;
    if (kb == 0) {
      if (cudaMemcpyAsync(CA + ma, LA + last * ma, sizeof(float2) * ma, cudaMemcpyDeviceToDevice,
                          st) != cudaSuccess ||
          cudaMemcpyAsync(CB + mb, LB + last * mb, sizeof(float2) * mb, cudaMemcpyDeviceToDevice,
                          st) != cudaSuccess)
        return cuda_fail(cudaGetLastError(), "affine carry copy");
      continue;
    }
    Operand cur{LA + last * ma, 0, 1};
    GOOM_TRY(lmme_call(cur, Operand{CA + kb * ma, 0, 1}, kNone, CA + (kb + 1) * ma, 0, 1, d, d, d,
                       lws, lws_bytes, st));
    GOOM_TRY(lmme_call(cur, Operand{CB + kb * mb, 0, 1}, Operand{LB + last * mb, 0, 1},
                       CB + (kb + 1) * mb, 0, 1, d, d, m, lws, lws_bytes, st));
  }
  // phase 3
  if (cudaMemcpyAsync(outA, LA, sizeof(float2) * ma * s, cudaMemcpyDeviceToDevice, st) !=
          cudaSuccess ||
      cudaMemcpyAsync(outB, LB, sizeof(float2) * mb * s, cudaMemcpyDeviceToDevice, st) !=
          cudaSuccess)
    return cuda_fail(cudaGetLastError(), "affine block-0 copy");
  if (T > s) {
    Operand cur{LA + s * ma, ma, 1};
    GOOM_TRY(lmme_call(cur, Operand{CA + ma, ma, s}, kNone, outA + s * ma, ma, T - s, d, d, d, lws,
                       lws_bytes, st));
    GOOM_TRY(lmme_call(cur, Operand{CB + mb, mb, s}, Operand{LB + s * mb, mb, 1}, outB + s * mb,
                       mb, T - s, d, d, m, lws, lws_bytes, st));
  }
  if (flags_out) GOOM_TRY(launch_flags_or_scan(flags_in, flags_out, T, st));
  return GOOM_OK;
}

}  // namespace goom

using namespace goom;

extern "C" {

size_t goom_scan_chain_workspace_size(int64_t T, int d, int block) {
  if (T < 1 || d < 1 || block < 1) return 0;
  return chain_workspace_bytes(T, d, block);
}

int goom_scan_chain_c64(const goom_c64* A, goom_c64* out, int64_t T, int d, int block,
                        const goom_c64* carry_in, void* ws, size_t ws_bytes, void* stream) {
  if (T < 1) return fail(GOOM_EINVAL, "scan of an empty sequence");
  if (block < 1) return fail(GOOM_EINVAL, "block_size must be >= 1");
  if (d < 1) return fail(GOOM_ESHAPE, "d must be >= 1");
  if (!A || !out) return fail(GOOM_EINVAL, "null pointer");
  return chain_scan(reinterpret_cast<const float2*>(A), reinterpret_cast<float2*>(out), T, d,
                    block, reinterpret_cast<const float2*>(carry_in), ws, ws_bytes,
                    as_stream(stream));
}

size_t goom_scan_affine_workspace_size(int64_t T, int d, int m, int block) {
  if (T < 1 || d < 1 || m < 1 || block < 1) return 0;
  return affine_workspace_bytes(T, d, m, block);
}

int goom_scan_affine_c64(const goom_c64* A, const goom_c64* B, const uint8_t* flags_in,
                         goom_c64* outA, goom_c64* outB, uint8_t* flags_out, int64_t T, int d,
                         int m, int block, void* ws, size_t ws_bytes, void* stream) {
  if (T < 1) return fail(GOOM_EINVAL, "scan of an empty sequence");
  if (block < 1) return fail(GOOM_EINVAL, "block_size must be >= 1");
  if (d < 1 || m < 1) return fail(GOOM_ESHAPE, "d and m must be >= 1");
  if (!A || !B || !outA || !outB) return fail(GOOM_EINVAL, "null pointer");
  return affine_scan(reinterpret_cast<const float2*>(A), reinterpret_cast<const float2*>(B),
                     flags_in, reinterpret_cast<float2*>(outA), reinterpret_cast<float2*>(outB),
                     flags_out, T, d, m, block, ws, ws_bytes, as_stream(stream));
}

}  // extern "C"
