// LMME dispatch: scale pre-pass + kernel-family selection + ABI entry points.
//   complex64 : tcgen05 3xTF32 (n, m % 128 == 0, k % 32 == 0) > SIMT small (<= 32) > SIMT tiled
//   complex128: SIMT FP64 small / tiled
#include <atomic>

#include "goom_internal.cuh"

namespace goom {

namespace {
std::atomic<int> g_backend{0};  // 0 auto, 1 SIMT, 2 tcgen05

inline int64_t distinct(int64_t stride, int64_t div, int64_t batch) {
  if (stride == 0 || batch == 0) return 1;
  return (batch - 1) / (div < 1 ? 1 : div) + 1;
}
inline size_t round_up(size_t x) { return (x + 255) & ~size_t(255); }

template <class R>
bool small_shape(int n, int k, int m) {
  return n <= 32 && k <= 32 && m <= 32;
}
bool whole_shape(int n, int k, int m) { return n <= 64 && k <= 64 && m <= 64; }
}  // namespace

int lmme_backend() { return g_backend.load(); }

template <class R>
size_t lmme_workspace_bytes(int64_t batch, int n, int k, int m, int64_t strideA, int64_t divA,
                            int64_t strideB, int64_t divB) {
  if (small_shape<R>(n, k, m) || whole_shape(n, k, m)) return 0;  // scales in-kernel
  return round_up(sizeof(R) * (size_t)distinct(strideA, divA, batch) * n) +
         round_up(sizeof(R) * (size_t)distinct(strideB, divB, batch) * m) + 256 /*phase flag*/;
}

template <class R>
int lmme_run(LmmeProblemT<R> p, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (p.batch == 0 || p.n == 0 || p.m == 0) return GOOM_OK;
  const int backend = g_backend.load();
  const bool small = small_shape<R>(p.n, p.k, p.m);
  if (small && !p.rowA.ptr) return lmme_simt_small<R>(p, s);
  if constexpr (sizeof(R) == 4) {
    // n = m = 64 (config 2): two products per tcgen05 tile, scales by the kernel's scale pass
    if (p.allow_duo && backend != 1 && !p.rowA.ptr && !p.colB.ptr && !p.emitRow && !p.emitCol) {
      const int rc = lmme_tc_duo(p, s);
      if (rc != GOOM_EUNSUPPORTED) return rc;
    }
  }
  // n, k, m <= 64 (and not a tcgen05 shape): one CTA per product, scales fused
  if (whole_shape(p.n, p.k, p.m) && !p.rowA.ptr &&
      !(sizeof(R) == 4 && backend != 1 && lmme_tc_eligible(p.n, p.k, p.m)))
    return lmme_simt_whole<R>(p, s);
  if constexpr (sizeof(R) == 4) {
    // n = m = 256 (config 2's HBM-bound shape): the pair kernel reduces the clamped scales
    // of its own A rows / B columns from HBM and its ring re-reads them from L2 (no pre-pass)
    // n = m = 128: the one-SM kernel reduces them in a scale pass through its ring
    if (backend != 1 && (!p.rowA.ptr || !p.colB.ptr) &&
        (lmme_tc2_fuse_scales(p.n, p.k, p.m) || lmme_tc1_fuse_scales(p.n, p.k, p.m))) {
      const int rc = lmme_tc(p, s);
      if (rc != GOOM_EUNSUPPORTED) return rc;
    }
  }
  if (!p.rowA.ptr || !p.colB.ptr) {
    size_t need = lmme_workspace_bytes<R>(p.batch, p.n, p.k, p.m, p.A.stride, p.A.div,
                                          p.B.stride, p.B.div);
    if (ws_bytes < need || (need && !ws))
      return fail(GOOM_EWORKSPACE, "lmme workspace too small (need " + std::to_string(need) +
                                       " bytes)");
    int64_t nA = distinct(p.A.stride, p.A.div, p.batch), nB = distinct(p.B.stride, p.B.div, p.batch);
    char* w = reinterpret_cast<char*>(ws);
    R* ra = reinterpret_cast<R*>(w);
    w += round_up(sizeof(R) * (size_t)nA * p.n);
    R* cb = reinterpret_cast<R*>(w);
    w += round_up(sizeof(R) * (size_t)nB * p.m);
    int* flag = nullptr;
    if (sizeof(R) == 4 && backend != 1 && lmme_tc_eligible(p.n, p.k, p.m)) {
      flag = reinterpret_cast<int*>(w);  // lets the tcgen05 transform take the 0 / pi fast path
      if (cudaMemsetAsync(flag, 0, sizeof(int), s) != cudaSuccess)
        return cuda_fail(cudaGetLastError(), "phase flag reset");
    }
    GOOM_TRY(launch_row_scales<R>(OperandT<Cx<R>>{p.A.ptr, p.A.stride, 1}, ra, nA, p.n, p.k, s, flag));
    GOOM_TRY(launch_col_scales<R>(OperandT<Cx<R>>{p.B.ptr, p.B.stride, 1}, cb, nB, p.k, p.m, s, flag));
    p.noncanon = flag;
    p.rowA = ScalesT<R>{ra, p.A.stride == 0 ? 0 : (int64_t)p.n, p.A.div};
    p.colB = ScalesT<R>{cb, p.B.stride == 0 ? 0 : (int64_t)p.m, p.B.div};
  }
  if constexpr (sizeof(R) == 4) {
    if (backend != 1 && lmme_tc_eligible(p.n, p.k, p.m)) {
      int rc = lmme_tc(p, s);
      if (rc != GOOM_EUNSUPPORTED) return rc;
    }
    if (backend == 2 && !small)
      return fail(GOOM_EUNSUPPORTED, "tcgen05 LMME needs n,m multiples of 128 and k of 32");
  }
  return lmme_simt_tiled<R>(p, s);
}

template size_t lmme_workspace_bytes<float>(int64_t, int, int, int, int64_t, int64_t, int64_t,
                                            int64_t);
template size_t lmme_workspace_bytes<double>(int64_t, int, int, int, int64_t, int64_t, int64_t,
                                             int64_t);
template int lmme_run<float>(LmmeProblemT<float>, void*, size_t, cudaStream_t);
template int lmme_run<double>(LmmeProblemT<double>, void*, size_t, cudaStream_t);

}  // namespace goom

using namespace goom;

namespace {

int check_lmme_args(const goom_operand& A, const goom_operand& B, const void* C, int64_t batch,
                    int n, int k, int m) {
  if (batch < 0) return fail(GOOM_EINVAL, "batch must be >= 0");
  if (n < 1 || k < 1 || m < 1) return fail(GOOM_ESHAPE, "lmme dimensions must be >= 1");
  if (batch > 0 && (!A.ptr || !B.ptr || !C)) return fail(GOOM_EINVAL, "null pointer");
  if (A.stride < 0 || B.stride < 0) return fail(GOOM_EINVAL, "negative stride");
  return GOOM_OK;
}

template <class R>
OperandT<Cx<R>> op(const goom_operand& o) {
  return OperandT<Cx<R>>{reinterpret_cast<const Cx<R>*>(o.ptr), o.stride, o.div < 1 ? 1 : o.div};
}

template <class R>
int lmme_entry(goom_operand A, goom_operand B, goom_operand D, void* C, int64_t strideC,
               int64_t batch, int n, int k, int m, void* ws, size_t ws_bytes, void* stream) {
  GOOM_TRY(check_lmme_args(A, B, C, batch, n, k, m));
  LmmeProblemT<R> p{};
  p.A = op<R>(A);
  p.B = op<R>(B);
  p.D = op<R>(D);
  p.C = reinterpret_cast<Cx<R>*>(C);
  p.strideC = strideC;
  p.batch = batch;
  p.n = n;
  p.k = k;
  p.m = m;
  p.rowA = ScalesT<R>{nullptr, 0, 1};
  p.colB = ScalesT<R>{nullptr, 0, 1};
  p.allow_duo = true;
  return lmme_run<R>(p, ws, ws_bytes, as_stream(stream));
}

const goom_operand kNoAddend{nullptr, 0, 1};

}  // namespace

extern "C" {

size_t goom_lmme_workspace_size(int64_t batch, int n, int k, int m) {
  return lmme_workspace_bytes<float>(batch, n, k, m, 1, 1, 1, 1);
}
size_t goom_lmme_workspace_size_c128(int64_t batch, int n, int k, int m) {
  return lmme_workspace_bytes<double>(batch, n, k, m, 1, 1, 1, 1);
}

int goom_lmme_c64(goom_operand A, goom_operand B, goom_c64* C, int64_t strideC, int64_t batch,
                  int n, int k, int m, void* ws, size_t ws_bytes, void* stream) {
  return lmme_entry<float>(A, B, kNoAddend, C, strideC, batch, n, k, m, ws, ws_bytes, stream);
}
int goom_lmme_gadd_c64(goom_operand A, goom_operand B, goom_operand D, goom_c64* C,
                       int64_t strideC, int64_t batch, int n, int k, int m, void* ws,
                       size_t ws_bytes, void* stream) {
  return lmme_entry<float>(A, B, D, C, strideC, batch, n, k, m, ws, ws_bytes, stream);
}
int goom_lmme_c128(goom_operand A, goom_operand B, goom_c128* C, int64_t strideC, int64_t batch,
                   int n, int k, int m, void* ws, size_t ws_bytes, void* stream) {
  return lmme_entry<double>(A, B, kNoAddend, C, strideC, batch, n, k, m, ws, ws_bytes, stream);
}
int goom_lmme_gadd_c128(goom_operand A, goom_operand B, goom_operand D, goom_c128* C,
                        int64_t strideC, int64_t batch, int n, int k, int m, void* ws,
                        size_t ws_bytes, void* stream) {
  return lmme_entry<double>(A, B, D, C, strideC, batch, n, k, m, ws, ws_bytes, stream);
}

int goom_lmme_scaled_c64(goom_operand A, const float* rowA, int64_t rowA_stride, goom_operand B,
                         const float* colB, int64_t colB_stride, goom_c64* C, int64_t strideC,
                         int64_t batch, int n, int k, int m, void* stream) {
  GOOM_TRY(check_lmme_args(A, B, C, batch, n, k, m));
  if (!rowA || !colB) return fail(GOOM_EINVAL, "null scale array");
  LmmeProblemT<float> p{};
  p.A = op<float>(A);
  p.B = op<float>(B);
  p.D = OperandT<float2>{nullptr, 0, 1};
  p.C = reinterpret_cast<float2*>(C);
  p.strideC = strideC;
  p.batch = batch;
  p.n = n;
  p.k = k;
  p.m = m;
  p.rowA = ScalesT<float>{rowA, rowA_stride, p.A.div};
  p.colB = ScalesT<float>{colB, colB_stride, p.B.div};
  return lmme_run<float>(p, nullptr, 0, as_stream(stream));
}

int goom_set_lmme_backend(int backend) {
  if (backend < 0 || backend > 2) return g_backend.load();
  return g_backend.exchange(backend);
}

}  // extern "C"
