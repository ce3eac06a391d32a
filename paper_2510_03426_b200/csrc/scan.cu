// Blocked prefix-scan engines over LMME combines (complex64 and complex128).
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
#include <atomic>
#include <cstdlib>

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

template <class R>
size_t lmme_ws(int64_t batch, int n, int m) {
  // worst case: every operand distinct
  return round_up(sizeof(R) * (size_t)batch * n) + round_up(sizeof(R) * (size_t)batch * m) + 256;
}

// C[b] = A(b) (x) B(b) (+) D(b)
template <class R>
int lmme_call(OperandT<Cx<R>> A, OperandT<Cx<R>> B, OperandT<Cx<R>> D, Cx<R>* C, int64_t strideC,
              int64_t batch, int n, int k, int m, void* ws, size_t ws_bytes, cudaStream_t s) {
  LmmeProblemT<R> p{};
  p.A = A;
  p.B = B;
  p.D = D;
  p.C = C;
  p.strideC = strideC;
  p.batch = batch;
  p.n = n;
  p.k = k;
  p.m = m;
  p.rowA = ScalesT<R>{nullptr, 0, 1};
  p.colB = ScalesT<R>{nullptr, 0, 1};
  return lmme_run<R>(p, ws, ws_bytes, s);
}

template <class C>
OperandT<C> opnd(const C* p, int64_t stride, int64_t div = 1) {
  return OperandT<C>{p, stride, div};
}

template <class C>
int copy_d2d(C* dst, const C* src, size_t count, cudaStream_t st, const char* what) {
  if (count && cudaMemcpyAsync(dst, src, sizeof(C) * count, cudaMemcpyDeviceToDevice, st) !=
                   cudaSuccess)
    return cuda_fail(cudaGetLastError(), what);
  return GOOM_OK;
}

// dst[k*pitch .. +width) = src[k*pitch .. +width) for k < rows (elements)
template <class C>
int copy_strided(C* dst, const C* src, size_t width, size_t pitch, size_t rows, cudaStream_t st,
                 const char* what) {
  if (cudaMemcpy2DAsync(dst, sizeof(C) * pitch, src, sizeof(C) * pitch, sizeof(C) * width, rows,
                        cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), what);
  return GOOM_OK;
}

}  // namespace

// The public complex64 chain scan keeps the reference's per-column clamped scales (Eq. 11,
// core.py:252-253) for every d: the tile-scaled engine (chain_ts.cu) is opt-in here
// (GOOM_CHAIN_TS=1) because its per-(row, 256-column block) format flushes entries more than
// ~e^87 below their block's largest (lmme_ts.cu header), where the reference is exact.
std::atomic<int> g_chain_engine{-1};  // -1: not read yet; 0 complex64 (exact); 1 tile-scaled
int chain_engine() {
  int v = g_chain_engine.load();
  if (v < 0) {
    const char* e = getenv("GOOM_CHAIN_TS");
    int want = (e && atoi(e) == 1) ? 1 : 0;
    g_chain_engine.compare_exchange_strong(v, want);
    v = g_chain_engine.load();
  }
  return v;
}
// GOOM_CHAIN_CTA=0 routes 32 < d <= 64 chains through the batched launches instead of the
// CTA-resident walks (bitwise-equality tests compare the two)
bool chain_cta_disabled() {
  static const bool off = [] {
    const char* e = getenv("GOOM_CHAIN_CTA");
    return e && atoi(e) == 0;
  }();
  return off;
}

bool chain_ts_path(int d) {
  return chain_engine() == 1 && lmme_backend() != 1 && lmme_ts_eligible(d, d, d);
}

template <class R>
size_t chain_workspace_bytes(int64_t T, int d, int block) {
  if (sizeof(R) == 4 && chain_ts_path(d)) return chain_c64_ts_workspace_bytes(T, d, block);
  int64_t s = block < T ? block : T;
  int64_t nb = (T + s - 1) / s;
  size_t mat = (size_t)d * d;
  return round_up(sizeof(Cx<R>) * mat * T) + round_up(sizeof(Cx<R>) * mat * (nb + 1)) +
         lmme_ws<R>(T, d, d) +
         // fused-scale tcgen05 path: row/col scales of leaves and local products, carries
         4 * round_up(sizeof(R) * (size_t)T * d) + 2 * round_up(sizeof(R) * (size_t)(nb + 1) * d) +
         256;
}

namespace {

// complex64 chain on the tcgen05 kernel with the scale reductions fused into the producing
// epilogues: only the leaves (and carry_in) get a scale pre-pass; every local product and
// carry arrives with its row / column maxima already reduced by the kernel that wrote it.
// Same tree and same LMME kernel as the generic path; only where the scales come from differs.
int chain_scan_tc(const float2* A, float2* out, int64_t T, int d, int64_t s, int64_t nb,
                  const float2* carry_in, float2* L, float2* Cx_, char* sbase, size_t sbytes,
                  cudaStream_t st) {
  using C = float2;
  const int64_t mat = (int64_t)d * d;
  Carve cv{sbase};
  float* rA = cv.take<float>((size_t)T * d);   // row scales of the leaves
  float* cA = cv.take<float>((size_t)T * d);   // column scales of the block-start leaves
  float* rL = cv.take<float>((size_t)T * d);   // emitted: row scales of L
  float* cL = cv.take<float>((size_t)T * d);   // emitted: column scales of L
  float* rC = cv.take<float>((size_t)(nb + 1) * d);
  float* cC = cv.take<float>((size_t)(nb + 1) * d);  // emitted: column scales of the carries
  int* flag = cv.take<int>(1);
  if (cv.off > sbytes) return fail(GOOM_EWORKSPACE, "chain scan workspace too small");
  (void)rC;
  if (cudaMemsetAsync(sbase, 0, cv.off, st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "scale workspace reset");
  // leaf pre-pass (also tells the kernel whether every phase is exactly 0 / pi)
  GOOM_TRY(launch_row_scales<float>(OperandT<C>{A, mat, 1}, rA, T, d, d, st, flag));
  GOOM_TRY(launch_col_scales<float>(OperandT<C>{A, s * mat, 1}, cA, nb, d, d, st, flag));
  // L[k*s] = A[k*s]: its scales are the leaf's
  if (cudaMemcpy2DAsync(rL, sizeof(float) * d * s, rA, sizeof(float) * d * s, sizeof(float) * d,
                        nb, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
      cudaMemcpy2DAsync(cL, sizeof(float) * d * s, cA, sizeof(float) * d, sizeof(float) * d, nb,
                        cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "block-start scales");
  if (carry_in)
    GOOM_TRY(launch_col_scales<float>(OperandT<C>{carry_in, 0, 1}, cC, 1, d, d, st, flag));

  auto run = [&](OperandT<C> a, ScalesT<float> ra, OperandT<C> b, ScalesT<float> cb, C* c,
                 int64_t strideC, int64_t batch, float* er, int64_t ers, float* ec,
                 int64_t ecs) {
    LmmeProblemT<float> p{};
    p.A = a;
    p.B = b;
    p.D = OperandT<C>{nullptr, 0, 1};
    p.C = c;
    p.strideC = strideC;
    p.batch = batch;
    p.n = p.k = p.m = d;
    p.rowA = ra;
    p.colB = cb;
    p.noncanon = flag;
    p.emitRow = er;
    p.emitRowStride = ers;
    p.emitCol = ec;
    p.emitColStride = ecs;
    return lmme_tc(p, st);
  };
  // phase 1: L[k*s+i] = A[k*s+i] (x) L[k*s+i-1], emitting the scales of L[k*s+i]
  for (int64_t i = 1; i < s; ++i) {
    int64_t cnt = (T - i + s - 1) / s;
    if (cnt <= 0) break;
    GOOM_TRY(run({A + i * mat, s * mat, 1}, {rA + i * d, s * d, 1}, {L + (i - 1) * mat, s * mat, 1},
                 {cL + (i - 1) * d, s * d, 1}, L + i * mat, s * mat, cnt, rL + i * d, s * d,
                 cL + i * d, s * d));
  }
  // phase 2: Cx[k+1] = L[last of block k] (x) Cx[k], emitting the carries' column scales
  for (int64_t kb = 0; kb + 1 < nb || (kb == 0 && !carry_in); ++kb) {
    int64_t last = kb * s + s - 1;
    if (kb == 0 && !carry_in) {
      GOOM_TRY(copy_d2d(Cx_ + mat, L + last * mat, mat, st, "chain carry copy"));
      GOOM_TRY(copy_d2d(cC + d, cL + last * d, d, st, "chain carry scale copy"));
      if (nb == 1) break;
      continue;
    }
    const C* prev = (kb == 0) ? carry_in : Cx_ + kb * mat;
    GOOM_TRY(run({L + last * mat, 0, 1}, {rL + last * d, 0, 1}, {prev, 0, 1}, {cC + kb * d, 0, 1},
                 Cx_ + (kb + 1) * mat, 0, 1, nullptr, 0, cC + (kb + 1) * d, 0));
  }
  // phase 3: out[b] = L[b] (x) Cx[b/s]
  if (carry_in) {
    GOOM_TRY(copy_d2d(Cx_, carry_in, mat, st, "chain carry-in copy"));
    GOOM_TRY(run({L, mat, 1}, {rL, d, 1}, {Cx_, mat, s}, {cC, d, s}, out, mat, T, nullptr, 0,
                 nullptr, 0));
  } else {
    GOOM_TRY(copy_d2d(out, L, (size_t)mat * s, st, "chain block-0 copy"));
    if (T > s)
      GOOM_TRY(run({L + s * mat, mat, 1}, {rL + s * d, d, 1}, {Cx_ + mat, mat, s}, {cC + d, d, s},
                   out + s * mat, mat, T - s, nullptr, 0, nullptr, 0));
  }
  return GOOM_OK;
}

bool fused_scale_path(const float2* A, const float2* carry_in, int d) {
  return lmme_backend() != 1 && lmme_tc_eligible(d, d, d) &&
         ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(carry_in)) & 15) == 0;
}

}  // namespace

template <class R>
int chain_scan(const Cx<R>* A, Cx<R>* out, int64_t T, int d, int block, const Cx<R>* carry_in,
               void* ws, size_t ws_bytes, cudaStream_t st) {
  using C = Cx<R>;
  const int64_t s = block < T ? block : T;
  const int64_t nb = (T + s - 1) / s;
  const int64_t mat = (int64_t)d * d;
  if (ws_bytes < chain_workspace_bytes<R>(T, d, block))
    return fail(GOOM_EWORKSPACE, "chain scan workspace too small");
  if constexpr (sizeof(R) == 4) {
    if (chain_ts_path(d))
      return chain_scan_c64_ts(A, out, T, d, block, carry_in, ws, ws_bytes, st);
  }
  Carve cv{reinterpret_cast<char*>(ws)};
  C* L = cv.take<C>((size_t)mat * T);
  C* Cx_ = cv.take<C>((size_t)mat * (nb + 1));
  void* lws = cv.base + cv.off;
  size_t lws_bytes = ws_bytes - cv.off;
  const OperandT<C> none{nullptr, 0, 1};

  // d <= 32: the warp-resident scan (scan_small.cu), same tree, three launches
  if (d <= 32) return chain_scan_small<R>(A, out, T, d, s, carry_in, L, Cx_, st);
  // 32 < d <= 64: the CTA-resident walks (scan_cta.cu), three launches
  if (chain_cta_eligible(d) && !chain_cta_disabled())
    return chain_scan_cta<R>(A, out, T, d, s, carry_in, L, Cx_, st);

  // phase 1: L[k*s] = A[k*s]; L[k*s+i] = A[k*s+i] (x) L[k*s+i-1]
  GOOM_TRY(copy_strided(L, A, mat, mat * s, nb, st, "chain phase-1 copy"));
  if constexpr (sizeof(R) == 4) {
    if (fused_scale_path(reinterpret_cast<const float2*>(A),
                         reinterpret_cast<const float2*>(carry_in), d))
      return chain_scan_tc(A, out, T, d, s, nb, carry_in, L, Cx_, reinterpret_cast<char*>(lws),
                           lws_bytes, st);
  }
  for (int64_t i = 1; i < s; ++i) {
    int64_t cnt = (T - i + s - 1) / s;  // blocks whose length exceeds i
    if (cnt <= 0) break;
    GOOM_TRY(lmme_call<R>(opnd(A + i * mat, s * mat), opnd<C>(L + (i - 1) * mat, s * mat), none,
                          L + i * mat, s * mat, cnt, d, d, d, lws, lws_bytes, st));
  }
  // phase 2: Cx[0] = carry_in; Cx[k+1] = L[last of block k] (x) Cx[k]
  for (int64_t kb = 0; kb + 1 < nb || (kb == 0 && !carry_in); ++kb) {
    int64_t last = kb * s + s - 1;
    if (kb == 0 && !carry_in) {
      GOOM_TRY(copy_d2d(Cx_ + mat, L + last * mat, mat, st, "chain carry copy"));
      if (nb == 1) break;
      continue;
    }
    const C* prev = (kb == 0) ? carry_in : Cx_ + kb * mat;
    GOOM_TRY(lmme_call<R>(opnd<C>(L + last * mat, 0), opnd(prev, 0), none, Cx_ + (kb + 1) * mat,
                          0, 1, d, d, d, lws, lws_bytes, st));
  }
  // phase 3: out[b] = L[b] (x) Cx[b/s]  (block 0 needs a carry only with carry_in)
  if (carry_in) {
    GOOM_TRY(copy_d2d(Cx_, carry_in, mat, st, "chain carry-in copy"));
    GOOM_TRY(lmme_call<R>(opnd<C>(L, mat), opnd<C>(Cx_, mat, s), none, out, mat, T, d, d, d, lws,
                          lws_bytes, st));
  } else {
    GOOM_TRY(copy_d2d(out, L, (size_t)mat * s, st, "chain block-0 copy"));
    if (T > s)
      GOOM_TRY(lmme_call<R>(opnd<C>(L + s * mat, mat), opnd<C>(Cx_ + mat, mat, s), none,
                            out + s * mat, mat, T - s, d, d, d, lws, lws_bytes, st));
  }
  return GOOM_OK;
}

template size_t chain_workspace_bytes<float>(int64_t, int, int);
template size_t chain_workspace_bytes<double>(int64_t, int, int);
template int chain_scan<float>(const float2*, float2*, int64_t, int, int, const float2*, void*,
                               size_t, cudaStream_t);
template int chain_scan<double>(const double2*, double2*, int64_t, int, int, const double2*,
                                void*, size_t, cudaStream_t);

namespace {

template <class R>
size_t affine_workspace_bytes(int64_t T, int d, int m, int block) {
  int64_t s = block < T ? block : T;
  int64_t nb = (T + s - 1) / s;
  const size_t e = sizeof(Cx<R>);
  return round_up(e * (size_t)d * d * T) + round_up(e * (size_t)d * m * T) +
         round_up(e * (size_t)d * d * (nb + 1)) + round_up(e * (size_t)d * m * (nb + 1)) +
         lmme_ws<R>(T, d, d > m ? d : m);
}

template <class R>
int affine_scan(const Cx<R>* A, const Cx<R>* B, const uint8_t* flags_in, Cx<R>* outA,
                Cx<R>* outB, uint8_t* flags_out, int64_t T, int d, int m, int block, void* ws,
                size_t ws_bytes, cudaStream_t st) {
  using C = Cx<R>;
  const int64_t s = block < T ? block : T;
  const int64_t nb = (T + s - 1) / s;
  const int64_t ma = (int64_t)d * d, mb = (int64_t)d * m;
  if (ws_bytes < affine_workspace_bytes<R>(T, d, m, block))
    return fail(GOOM_EWORKSPACE, "affine scan workspace too small");
  Carve cv{reinterpret_cast<char*>(ws)};
  C* LA = cv.take<C>((size_t)ma * T);
  C* LB = cv.take<C>((size_t)mb * T);
  C* CA = cv.take<C>((size_t)ma * (nb + 1));
  C* CB = cv.take<C>((size_t)mb * (nb + 1));
  void* lws = cv.base + cv.off;
  size_t lws_bytes = ws_bytes - cv.off;
  const OperandT<C> none{nullptr, 0, 1};

  GOOM_TRY(copy_strided(LA, A, ma, ma * s, nb, st, "affine phase-1 copy"));
  GOOM_TRY(copy_strided(LB, B, mb, mb * s, nb, st, "affine phase-1 copy"));
  // phase 1 (combine_affine, scan.py:173-178): A slot, then the fused bias slot
  for (int64_t i = 1; i < s; ++i) {
    int64_t cnt = (T - i + s - 1) / s;
    if (cnt <= 0) break;
    auto cur = opnd(A + i * ma, s * ma);
    GOOM_TRY(lmme_call<R>(cur, opnd<C>(LA + (i - 1) * ma, s * ma), none, LA + i * ma, s * ma, cnt,
                          d, d, d, lws, lws_bytes, st));
    GOOM_TRY(lmme_call<R>(cur, opnd<C>(LB + (i - 1) * mb, s * mb), opnd(B + i * mb, s * mb),
                          LB + i * mb, s * mb, cnt, d, d, m, lws, lws_bytes, st));
  }
  // phase 2: carries of blocks 0 .. nb-2
  for (int64_t kb = 0; kb + 1 < nb; ++kb) {
    int64_t last = kb * s + s - 1;
    if (kb == 0) {
      GOOM_TRY(copy_d2d(CA + ma, LA + last * ma, ma, st, "affine carry copy"));
      GOOM_TRY(copy_d2d(CB + mb, LB + last * mb, mb, st, "affine carry copy"));
      continue;
    }
    auto cur = opnd<C>(LA + last * ma, 0);
    GOOM_TRY(lmme_call<R>(cur, opnd<C>(CA + kb * ma, 0), none, CA + (kb + 1) * ma, 0, 1, d, d, d,
                          lws, lws_bytes, st));
    GOOM_TRY(lmme_call<R>(cur, opnd<C>(CB + kb * mb, 0), opnd<C>(LB + last * mb, 0),
                          CB + (kb + 1) * mb, 0, 1, d, d, m, lws, lws_bytes, st));
  }
  // phase 3
  GOOM_TRY(copy_d2d(outA, LA, (size_t)ma * s, st, "affine block-0 copy"));
  GOOM_TRY(copy_d2d(outB, LB, (size_t)mb * s, st, "affine block-0 copy"));
  if (T > s) {
    auto cur = opnd<C>(LA + s * ma, ma);
    GOOM_TRY(lmme_call<R>(cur, opnd<C>(CA + ma, ma, s), none, outA + s * ma, ma, T - s, d, d, d,
                          lws, lws_bytes, st));
    GOOM_TRY(lmme_call<R>(cur, opnd<C>(CB + mb, mb, s), opnd<C>(LB + s * mb, mb), outB + s * mb,
                          mb, T - s, d, d, m, lws, lws_bytes, st));
  }
  if (flags_out) GOOM_TRY(launch_flags_or_scan(flags_in, flags_out, T, st));
  return GOOM_OK;
}

int check_scan(int64_t T, int block, int d, int m) {
  if (T < 1) return fail(GOOM_EINVAL, "scan of an empty sequence");
  if (block < 1) return fail(GOOM_EINVAL, "block_size must be >= 1");
  if (d < 1 || m < 1) return fail(GOOM_ESHAPE, "d and m must be >= 1");
  return GOOM_OK;
}

template <class R>
int chain_entry(const void* A, void* out, int64_t T, int d, int block, const void* carry_in,
                void* ws, size_t ws_bytes, void* stream) {
  GOOM_TRY(check_scan(T, block, d, 1));
  if (!A || !out) return fail(GOOM_EINVAL, "null pointer");
  return chain_scan<R>(reinterpret_cast<const Cx<R>*>(A), reinterpret_cast<Cx<R>*>(out), T, d,
                       block, reinterpret_cast<const Cx<R>*>(carry_in), ws, ws_bytes,
                       as_stream(stream));
}

template <class R>
int affine_entry(const void* A, const void* B, const uint8_t* flags_in, void* outA, void* outB,
                 uint8_t* flags_out, int64_t T, int d, int m, int block, void* ws,
                 size_t ws_bytes, void* stream) {
  GOOM_TRY(check_scan(T, block, d, m));
  if (!A || !B || !outA || !outB) return fail(GOOM_EINVAL, "null pointer");
  return affine_scan<R>(reinterpret_cast<const Cx<R>*>(A), reinterpret_cast<const Cx<R>*>(B),
                        flags_in, reinterpret_cast<Cx<R>*>(outA), reinterpret_cast<Cx<R>*>(outB),
                        flags_out, T, d, m, block, ws, ws_bytes, as_stream(stream));
}

}  // namespace
}  // namespace goom

using namespace goom;

extern "C" {

size_t goom_scan_chain_workspace_size(int64_t T, int d, int block) {
  if (T < 1 || d < 1 || block < 1) return 0;
  return chain_workspace_bytes<float>(T, d, block);
}
size_t goom_scan_chain_workspace_size_c128(int64_t T, int d, int block) {
  if (T < 1 || d < 1 || block < 1) return 0;
  return chain_workspace_bytes<double>(T, d, block);
}
int goom_scan_chain_c64(const goom_c64* A, goom_c64* out, int64_t T, int d, int block,
                        const goom_c64* carry_in, void* ws, size_t ws_bytes, void* stream) {
  return chain_entry<float>(A, out, T, d, block, carry_in, ws, ws_bytes, stream);
}
int goom_scan_chain_c128(const goom_c128* A, goom_c128* out, int64_t T, int d, int block,
                         const goom_c128* carry_in, void* ws, size_t ws_bytes, void* stream) {
  return chain_entry<double>(A, out, T, d, block, carry_in, ws, ws_bytes, stream);
}

size_t goom_scan_affine_workspace_size(int64_t T, int d, int m, int block) {
  if (T < 1 || d < 1 || m < 1 || block < 1) return 0;
  return affine_workspace_bytes<float>(T, d, m, block);
}
size_t goom_scan_affine_workspace_size_c128(int64_t T, int d, int m, int block) {
  if (T < 1 || d < 1 || m < 1 || block < 1) return 0;
  return affine_workspace_bytes<double>(T, d, m, block);
}
int goom_scan_affine_c64(const goom_c64* A, const goom_c64* B, const uint8_t* flags_in,
                         goom_c64* outA, goom_c64* outB, uint8_t* flags_out, int64_t T, int d,
                         int m, int block, void* ws, size_t ws_bytes, void* stream) {
  return affine_entry<float>(A, B, flags_in, outA, outB, flags_out, T, d, m, block, ws, ws_bytes,
                             stream);
}
int goom_scan_affine_c128(const goom_c128* A, const goom_c128* B, const uint8_t* flags_in,
                          goom_c128* outA, goom_c128* outB, uint8_t* flags_out, int64_t T, int d,
                          int m, int block, void* ws, size_t ws_bytes, void* stream) {
  return affine_entry<double>(A, B, flags_in, outA, outB, flags_out, T, d, m, block, ws, ws_bytes,
                              stream);
}

}  // extern "C"

extern "C" int goom_set_chain_engine(int engine) {
  goom::chain_engine();  // settle the environment default first
  if (engine < 0 || engine > 1) return goom::g_chain_engine.load();
  return goom::g_chain_engine.exchange(engine);
}
