// LMME dispatch: scale pre-pass + kernel-family selection + ABI entry points.
#include <atomic>

#include "goom_internal.cuh"

namespace goom {

namespace {
std::atomic<int> g_backend{0};  // 0 auto, 1 SIMT, 2 tcgen05

inline int64_t distinct(const Operand& o, int64_t batch) {
  if (o.stride == 0 || batch == 0) return 1;
  return (batch - 1) / o.div + 1;
}
inline size_t round_up(size_t x) { return (x + 255) & ~size_t(255); }
}  // namespace

int lmme_backend() { return g_backend.load(); }

size_t lmme_workspace_bytes(int64_t batch, int n, int k, int m, const Operand& A,
                            const Operand& B) {
  (void)k;
  if (n <= 32 && k <= 32 && m <= 32 && g_backend.load() != 2) return 0;  // small kernel: in-kernel
  return round_up(sizeof(float) * (size_t)distinct(A, batch) * n) +
         round_up(sizeof(float) * (size_t)distinct(B, batch) * m);
}

int lmme_run(LmmeProblem p, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (p.batch == 0 || p.n == 0 || p.m == 0) return GOOM_OK;
  const int backend = g_backend.load();
  const bool small = p.n <= 32 && p.k <= 32 && p.m <= 32;
  if (small && backend != 2 && !p.rowA.ptr) return lmme_simt_small(p, s);
  if (!p.rowA.ptr || !p.colB.ptr) {
    size_t need = lmme_workspace_bytes(p.batch, p.n, p.k, p.m, p.A, p.B);
    if (ws_bytes < need || (need && !ws))
      return fail(GOOM_EWORKSPACE, "lmme workspace too small (need " + std::to_string(need) +
                                       " bytes)");
    int64_t nA = distinct(p.A, p.batch), nB = distinct(p.B, p.batch);
    float* ra = reinterpret_cast<float*>(ws);
    float* cb = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) +
                                         round_up(sizeof(float) * (size_t)nA * p.n));
    GOOM_TRY(launch_row_scales(Operand{p.A.ptr, p.A.stride, 1}, ra, nA, p.n, p.k, s));
    GOOM_TRY(launch_col_scales(Operand{p.B.ptr, p.B.stride, 1}, cb, nB, p.k, p.m, s));
    p.rowA = Scales{ra, p.A.stride == 0 ? 0 : (int64_t)p.n, p.A.div};
    p.colB = Scales{cb, p.B.stride == 0 ? 0 : (int64_t)p.m, p.B.div};
  }
  if (backend != 1 && lmme_tc_eligible(p.n, p.k, p.m)) {
    int rc = lmme_tc(p, s);
    if (rc != GOOM_EUNSUPPORTED) return rc;
  }
  if (backend == 2 && !lmme_tc_eligible(p.n, p.k, p.m) && !small)
    return fail(GOOM_EUNSUPPORTED, "tcgen05 LMME needs n,m multiples of 128 and k of 32");
  return lmme_simt_tiled(p, s);
}

}  // namespace goom

using namespace goom;

namespace {
int check_lmme_args(const goom_operand& A, const goom_operand& B, const goom_c64* C,
                    int64_t batch, int n, int k, int m) {
  if (batch < 0) return fail(GOOM_EINVAL, "batch must be >= 0");
  if (n < 1 || k < 1 || m < 1) return fail(GOOM_ESHAPE, "lmme dimensions must be >= 1");
  if (batch > 0 && (!A.ptr || !B.ptr || !C)) return fail(GOOM_EINVAL, "null pointer");
  if (A.stride < 0 || B.stride < 0) return fail(GOOM_EINVAL, "negative stride");
  return GOOM_OK;
}
}  // namespace

extern "C" {

size_t goom_lmme_workspace_size(int64_t batch, int n, int k, int m) {
  Operand a{nullptr, 1, 1}, b{nullptr, 1, 1};
  return lmme_workspace_bytes(batch, n, k, m, a, b);
}

int goom_lmme_c64(goom_operand A, goom_operand B, goom_c64* C, int64_t strideC, int64_t batch,
                  int n, int k, int m, void* ws, size_t ws_bytes, void* stream) {
  goom_operand D{nullptr, 0, 1};
  return goom_lmme_gadd_c64(A, B, D, C, strideC, batch, n, k, m, ws, ws_bytes, stream);
}

int goom_lmme_gadd_c64(goom_operand A, goom_operand B, goom_operand D, goom_c64* C,
                       int64_t strideC, int64_t batch, int n, int k, int m, void* ws,
                       size_t ws_bytes, void* stream) {
  GOOM_TRY(check_lmme_args(A, B, C, batch, n, k, m));
  LmmeProblem p{};
  p.A = make_operand(A.ptr, A.stride, A.div);
  p.B = make_operand(B.ptr, B.stride, B.div);
  p.D = make_operand(D.ptr, D.stride, D.div);
  p.C = reinterpret_cast<float2*>(C);
  p.strideC = strideC;
  p.batch = batch;
  p.n = n;
  p.k = k;
  p.m = m;
  p.rowA = Scales{nullptr, 0, 1};
  p.colB = Scales{nullptr, 0, 1};
  return lmme_run(p, ws, ws_bytes, as_stream(stream));
}

int goom_set_lmme_backend(int backend) {
  if (backend < 0 || backend > 2) return g_backend.load();
  return g_backend.exchange(backend);
}

}  // extern "C"
