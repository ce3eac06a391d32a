// Chain scan over tile-scaled fp32 matrices (lmme_ts.cu) for d a multiple of 256.
//
// Same two-level tree as the reference's _scan_affine_stack A slot (scan.py:181-214) and
// as chain_scan (scan.cu) for the same block size s:
//   phase 1  L[ks+i] = A[ks+i] (x) L[ks+i-1], batched over blocks (s-1 launches);
//   phase 2  Cx[k+1] = L[last of block k] (x) Cx[k] (sequential fold; Cx[0] = carry-in, or
//            the identity when there is none, so every prefix is L_t (x) Cx[k]);
//   phase 3  P_t = L_t (x) Cx[t / s], one batched launch, written as complex64 GOOMs (the
//            public scan) or reduced on the fly to per-prefix digests (the long-chain
//            harness: 2 TiB of d = 512 prefixes are never stored).
// Cx[nb] = P_{T-1} is the carry-out of a window. Between phases every matrix stays
// tile-scaled: no exp/log per element except the leaf import and the final export.
#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>

#include "goom_internal.cuh"

namespace goom {

namespace {

inline size_t rup(size_t x) { return (x + 255) & ~size_t(255); }

struct TsBuf {  // T tile-scaled d x d matrices, contiguous
  float* U;
  float* q;
  uint32_t* G;
  int d, nJ;
  TsIn in(int64_t first = 0, int64_t stride_mats = 1, int64_t div = 1) const {
    const int64_t mat = (int64_t)d * d, qm = (int64_t)d * nJ;
    return TsIn{U + first * mat, q + first * qm, G + first * nJ, stride_mats * mat,
                stride_mats * qm, stride_mats * nJ, div};
  }
  TsOut out(int64_t first = 0, int64_t stride_mats = 1) const {
    const int64_t mat = (int64_t)d * d, qm = (int64_t)d * nJ;
    return TsOut{U + first * mat, q + first * qm, G + first * nJ, stride_mats * mat,
                 stride_mats * qm, stride_mats * nJ};
  }
};

size_t ts_bytes(int64_t mats, int d) {
  const int nJ = d / 256;
  return rup(sizeof(float) * (size_t)mats * d * d) + rup(sizeof(float) * (size_t)mats * d * nJ) +
         rup(sizeof(uint32_t) * (size_t)mats * nJ);
}

struct Carve {
  char* base;
  size_t off = 0;
  template <class X>
  X* take(size_t count) {
    X* p = reinterpret_cast<X*>(base + off);
    off += rup(sizeof(X) * count);
    return p;
  }
  TsBuf ts(int64_t mats, int d) {
    const int nJ = d / 256;
    TsBuf b;
    b.d = d;
    b.nJ = nJ;
    b.U = take<float>((size_t)mats * d * d);
    b.q = take<float>((size_t)mats * d * nJ);
    b.G = take<uint32_t>((size_t)mats * nJ);
    return b;
  }
};

int copy_ts(const TsBuf& dst, int64_t dfirst, const TsBuf& src, int64_t sfirst, int64_t count,
            int64_t sstride, cudaStream_t st, int64_t dstride = 0) {
  // count matrices src[sfirst + i*sstride] -> dst[dfirst + i*dstride] (dstride 0: = sstride)
  if (dstride == 0) dstride = sstride;
  const size_t mat = (size_t)src.d * src.d, qm = (size_t)src.d * src.nJ;
  const size_t w[3] = {mat * 4, qm * 4, (size_t)src.nJ * 4};
  const char* s[3] = {reinterpret_cast<const char*>(src.U + sfirst * mat),
                      reinterpret_cast<const char*>(src.q + sfirst * qm),
                      reinterpret_cast<const char*>(src.G + sfirst * src.nJ)};
  char* d[3] = {reinterpret_cast<char*>(dst.U + dfirst * mat),
                reinterpret_cast<char*>(dst.q + dfirst * qm),
                reinterpret_cast<char*>(dst.G + dfirst * dst.nJ)};
  for (int i = 0; i < 3; ++i)
    if (cudaMemcpy2DAsync(d[i], w[i] * dstride, s[i], w[i] * sstride, w[i], count,
                          cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return cuda_fail(cudaGetLastError(), "tile-scaled copy");
  return GOOM_OK;
}

int lmme_ts_call(TsIn a, TsIn b, int kind, float2* C, int64_t strideC, TsOut T, float4* parts,
                 int64_t batch, int d, cudaStream_t st) {
  TsProblem p{};
  p.A = a;
  p.B = b;
  p.kind = kind;
  p.C = C;
  p.strideC = strideC;
  p.T = T;
  p.parts = parts;
  p.batch = batch;
  p.n = p.k = p.m = d;
  return lmme_ts(p, st);
}

}  // namespace

// Per-phase launch timing inside real runs (bench.py's roofline: every kernel of the step
// measured in the timed region, on the stream it runs on): when enabled, each phase of a
// window (0 leaf generation, 1 local products, 2 block-carry tree, 3 digest / prefix
// output) is bracketed by a pair of CUDA events; the totals are read back later.
struct PhaseLog {
  std::mutex mu;
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[kPhases];
  std::vector<int64_t> units[kPhases];
};
static PhaseLog& phase_log() {
  static PhaseLog log;
  return log;
}
PhaseTimer::PhaseTimer(cudaStream_t s, int phase, int64_t units) : st(s), ph(phase), n(units) {
  PhaseLog& log = phase_log();
  std::lock_guard<std::mutex> lock(log.mu);
  if (!log.on) return;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
}
void PhaseTimer::stop() {
  if (!a) return;
  cudaEventRecord(b, st);
  PhaseLog& log = phase_log();
  std::lock_guard<std::mutex> lock(log.mu);
  log.ev[ph].emplace_back(a, b);
  log.units[ph].push_back(n);
  a = nullptr;
}

namespace {

}  // namespace

size_t chain_ts_workspace_bytes(int64_t T, int d, int block, bool leaves_given_ts) {
  const int64_t s = block < T ? block : T;
  const int64_t nb = (T + s - 1) / s;
  return (leaves_given_ts ? 0 : ts_bytes(T, d)) + ts_bytes(T, d) + 2 * ts_bytes(nb + 1, d) +
         rup(sizeof(float2) * (size_t)d * d) +                       // identity (complex64)
         rup(sizeof(float4) * (size_t)T * (d / 32) * (d / 256)) +    // digest partials
         rup(sizeof(uint32_t) * (size_t)nb * (d / 256)) +            // phase-1 counters
         1024;
}

struct ChainWs {
  TsBuf L, Cx, Cy;
  float2* ident;
  float4* parts;
  uint32_t* done;  // chained phase-1 counters, nb x d / 256
  int64_t s, nb;
};

// GOOM_CHAIN_PERSISTENT=1 runs phase 1 as ONE persistent launch (lmme_ts chained mode)
// instead of s - 1 batched launches. Off by default: under the B200's power cap the
// launches' fill / drain bubbles cost no throughput (the clock rises in them) and the
// persistent form measured 1-3% slower on phase 1 (profiles/r1_chain_persistent_ab.txt).
bool chain_persistent() {
  static const bool v = [] {
    const char* e = std::getenv("GOOM_CHAIN_PERSISTENT");
    return e && e[0] == '1';
  }();
  return v;
}

// carve the window workspace (the same layout for every stage, so a caller can keep it
// between chain_local and chain_finish)
int chain_ws(int64_t T, int d, int block, char* ws, size_t ws_bytes, ChainWs& w) {
  w.s = block < T ? block : T;
  w.nb = (T + w.s - 1) / w.s;
  Carve cv{ws};
  w.L = cv.ts(T, d);
  w.Cx = cv.ts(w.nb + 1, d);
  w.Cy = cv.ts(w.nb + 1, d);  // Kogge-Stone ping-pong buffer / carried carries
  w.ident = cv.take<float2>((size_t)d * d);
  w.parts = cv.take<float4>((size_t)T * (d / 32) * (d / 256));
  w.done = cv.take<uint32_t>((size_t)w.nb * (d / 256));
  if (cv.off > ws_bytes) return fail(GOOM_EWORKSPACE, "tile-scaled chain workspace too small");
  return GOOM_OK;
}

// phases 1 and 2: local products L and the block carries Cx[0..nb] (Cx[0] = carry-in or I,
// Cx[nb] = the window's last prefix); carry-independent when carry_in is null
int chain_local(const TsBuf& A, int64_t T, int d, int block, const TsBuf* carry_in, char* ws,
                size_t ws_bytes, cudaStream_t st, bool tree_carries) {
  ChainWs w;
  GOOM_TRY(chain_ws(T, d, block, ws, ws_bytes, w));
  const int64_t s = w.s, nb = w.nb;
  TsBuf &L = w.L, &Cx = w.Cx, &Cy = w.Cy;
  float2* ident = w.ident;
  const int nJ = d / 256;
  // every G slot that an epilogue max-reduces starts at "unset" (0)
  if (cudaMemsetAsync(L.G, 0, sizeof(uint32_t) * (size_t)T * nJ, st) != cudaSuccess ||
      cudaMemsetAsync(Cx.G, 0, sizeof(uint32_t) * (size_t)(nb + 1) * nJ, st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "tile-scaled G reset");
  // Cx[0]: carry-in or the identity
  if (carry_in) {
    GOOM_TRY(copy_ts(Cx, 0, *carry_in, 0, 1, 1, st));
  } else {
    GOOM_TRY(launch_identity<float>(ident, 1, d, (int64_t)d * d, st));
    GOOM_TRY(launch_goom_to_ts(ident, 0, Cx.out(0), 1, d, d, st));
  }
  // phase 1
  PhaseTimer t1(st, 1, T - nb);
  GOOM_TRY(copy_ts(L, 0, A, 0, nb, s, st));  // L[ks] = A[ks]
  if (s > 1 && T % s == 0 && chain_persistent()) {
    // every step of every block chain in ONE persistent launch: tiles run step-major and
    // wait on per-(block, column tile) completion counters instead of kernel boundaries
    uint32_t* done = w.done;
    if (cudaMemsetAsync(done, 0, sizeof(uint32_t) * (size_t)nb * nJ, st) != cudaSuccess)
      return cuda_fail(cudaGetLastError(), "chain counters reset");
    TsProblem p{};
    p.A = A.in(0, 1);
    p.B = L.in(0, 1);
    p.kind = kTsOutTs;
    p.T = L.out(0, 1);
    p.batch = nb;
    p.n = p.k = p.m = d;
    p.chain_s = (int)s;
    p.chain_T = T;
    p.chain_done = done;
    GOOM_TRY(lmme_ts(p, st));
  } else
  for (int64_t i = 1; i < s; ++i) {
    const int64_t cnt = (T - i + s - 1) / s;
    if (cnt <= 0) break;
    GOOM_TRY(lmme_ts_call(A.in(i, s), L.in(i - 1, s), kTsOutTs, nullptr, 0, L.out(i, s), nullptr,
                          cnt, d, st));
  }
  t1.stop();
  // phase 2: Cx[k+1] = L[last of block k] (x) Cx[k]
  int64_t p2 = 0;  // products of the carry tree
  if (tree_carries && nb > 1)
    for (int64_t h = 1; h < nb; h <<= 1) p2 += nb - h;
  else
    p2 = carry_in ? nb : nb - 1;
  PhaseTimer t2(st, 2, p2 + (tree_carries && nb > 1 && carry_in ? 1 : 0));
  if (tree_carries && nb > 1) {
    // X[k] (block k's carry-out, stored at Cx[k+1]) starts as the block total L[last of k]
    // (block 0: L[s-1] (x) Cx[0]); level j: X[k] <- X[k] (x) X[k - 2^j] for k >= 2^j
    if (cudaMemsetAsync(Cy.G, 0, sizeof(uint32_t) * (size_t)(nb + 1) * nJ, st) != cudaSuccess)
      return cuda_fail(cudaGetLastError(), "tile-scaled G reset");
    GOOM_TRY(copy_ts(Cx, 1, L, s - 1, nb - 1, s, st, 1));  // totals of blocks 0 .. nb-2
    const int64_t lastT = T - 1;                          // block nb-1 may be partial
    GOOM_TRY(copy_ts(Cx, nb, L, lastT, 1, 1, st));
    if (carry_in) {
      GOOM_TRY(lmme_ts_call(L.in(s - 1, 0), Cx.in(0, 0), kTsOutTs, nullptr, 0, Cy.out(1, 0),
                            nullptr, 1, d, st));
      GOOM_TRY(copy_ts(Cx, 1, Cy, 1, 1, 1, st));
    }
    TsBuf* X = &Cx;
    TsBuf* Y = &Cy;
    for (int64_t h = 1; h < nb; h <<= 1) {
      // Y[1 + k] = X[1 + k] (x) X[1 + k - h] for k >= h; Y[1 + k] = X[1 + k] below
      if (cudaMemsetAsync(Y->G + (1 + h) * nJ, 0, sizeof(uint32_t) * (size_t)(nb - h) * nJ, st) !=
          cudaSuccess)
        return cuda_fail(cudaGetLastError(), "tile-scaled G reset");
      GOOM_TRY(lmme_ts_call(X->in(1 + h, 1), X->in(1, 1), kTsOutTs, nullptr, 0, Y->out(1 + h, 1),
                            nullptr, nb - h, d, st));
      GOOM_TRY(copy_ts(*Y, 1, *X, 1, h, 1, st));
      TsBuf* tmp = X;
      X = Y;
      Y = tmp;
    }
    if (X != &Cx) GOOM_TRY(copy_ts(Cx, 1, *X, 1, nb, 1, st));
  } else {
    for (int64_t kb = 0; kb < nb; ++kb) {
      const int64_t last = kb * s + s - 1 < T ? kb * s + s - 1 : T - 1;
      if (kb == 0 && !carry_in) {
        GOOM_TRY(copy_ts(Cx, 1, L, last, 1, 1, st));
        continue;
      }
      GOOM_TRY(lmme_ts_call(L.in(last, 0), Cx.in(kb, 0), kTsOutTs, nullptr, 0,
                            Cx.out(kb + 1, 0), nullptr, 1, d, st));
    }
  }
  t2.stop();
  return GOOM_OK;
}

// phase 3 (+ optional right carry applied to every block carry first):
// P_t = L_t (x) (Cx[t / s] (x) carry); the carry-out is the last prefix
int chain_finish(int64_t T, int d, int block, const TsBuf* carry, float2* out, float4* digests,
                 TsBuf* carry_out, char* ws, size_t ws_bytes, cudaStream_t st) {
  ChainWs w;
  GOOM_TRY(chain_ws(T, d, block, ws, ws_bytes, w));
  const int64_t s = w.s, nb = w.nb;
  const int nJ = d / 256;
  if (carry) {  // Cx[k] <- Cx[k] (x) carry, one batched launch (Cx[0] = I -> carry)
    if (cudaMemsetAsync(w.Cy.G, 0, sizeof(uint32_t) * (size_t)(nb + 1) * nJ, st) != cudaSuccess)
      return cuda_fail(cudaGetLastError(), "tile-scaled G reset");
    GOOM_TRY(lmme_ts_call(w.Cx.in(0, 1), carry->in(0, 0), kTsOutTs, nullptr, 0, w.Cy.out(0, 1),
                          nullptr, nb + 1, d, st));
    GOOM_TRY(copy_ts(w.Cx, 0, w.Cy, 0, nb + 1, 1, st));
  }
  if (out)
    GOOM_TRY(lmme_ts_call(w.L.in(0, 1), w.Cx.in(0, 1, s), kTsOutGoom, out, (int64_t)d * d,
                          TsOut{}, nullptr, T, d, st));
  if (digests) {
    PhaseTimer timer(st, 3, T);
    GOOM_TRY(lmme_ts_call(w.L.in(0, 1), w.Cx.in(0, 1, s), kTsOutDigest, nullptr, 0, TsOut{},
                          w.parts, T, d, st));
    timer.stop();
    GOOM_TRY(launch_digest_reduce(w.parts, (d / 32) * nJ, digests, T, st));
  }
  if (carry_out) GOOM_TRY(copy_ts(*carry_out, 0, w.Cx, nb, 1, 1, st));
  return GOOM_OK;
}

// A (tile-scaled leaves, T of them) -> out (complex64 prefixes) or digests (T float4);
// carry_in / carry_out tile-scaled (may be null). tree_carries: phase 2 as a Kogge-Stone
// scan of the block totals (ceil(log2 nb) batched launches, ~nb log2 nb products) instead
// of the reference's sequential fold (nb dependent single-product launches, each on 8 of
// the 148 SMs at d = 512); a different but fixed combine tree, deterministic per (T, block).
int chain_scan_ts(const TsBuf& A, int64_t T, int d, int block, const TsBuf* carry_in,
                  float2* out, float4* digests, TsBuf* carry_out, char* ws, size_t ws_bytes,
                  cudaStream_t st, bool tree_carries) {
  GOOM_TRY(chain_local(A, T, d, block, carry_in, ws, ws_bytes, st, tree_carries));
  return chain_finish(T, d, block, nullptr, out, digests, carry_out, ws, ws_bytes, st);
}

// complex64 leaves -> tile-scaled -> chain_scan_ts (the public chain scan for d % 256 == 0)
int chain_scan_c64_ts(const float2* A, float2* out, int64_t T, int d, int block,
                      const float2* carry_in, void* ws, size_t ws_bytes, cudaStream_t st) {
  Carve cv{reinterpret_cast<char*>(ws)};
  TsBuf At = cv.ts(T, d);
  TsBuf Ci = cv.ts(1, d);
  const int nJ = d / 256;
  if (cudaMemsetAsync(At.G, 0, sizeof(uint32_t) * (size_t)T * nJ, st) != cudaSuccess ||
      cudaMemsetAsync(Ci.G, 0, sizeof(uint32_t) * nJ, st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "tile-scaled G reset");
  GOOM_TRY(launch_goom_to_ts(A, (int64_t)d * d, At.out(0), T, d, d, st));
  if (carry_in) GOOM_TRY(launch_goom_to_ts(carry_in, 0, Ci.out(0), 1, d, d, st));
  if (cv.off > ws_bytes) return fail(GOOM_EWORKSPACE, "chain workspace too small");
  return chain_scan_ts(At, T, d, block, carry_in ? &Ci : nullptr, out, nullptr, nullptr,
                       cv.base + cv.off, ws_bytes - cv.off, st, /*tree_carries=*/false);
}

size_t chain_c64_ts_workspace_bytes(int64_t T, int d, int block) {
  return ts_bytes(T, d) + ts_bytes(1, d) + chain_ts_workspace_bytes(T, d, block, true);
}

}  // namespace goom

using namespace goom;

namespace {
TsBuf ts_of(float* U, float* q, uint32_t* G, int d) {
  TsBuf b;
  b.U = U;
  b.q = q;
  b.G = G;
  b.d = d;
  b.nJ = d / 256;
  return b;
}
}  // namespace

extern "C" {

// Per-phase launch timing (profiling aid for bench.py): enable != 0 starts a fresh log;
// goom_chain_ts_phase_stats synchronises the logged events of one phase and returns its
// bracketed launches, their total milliseconds and total units (products; leaf matrices for
// phase 0). The phase3 pair is the phase-3 special case, kept for existing callers.
void goom_chain_ts_phase3_timing(int enable) {
  PhaseLog& log = phase_log();
  std::lock_guard<std::mutex> lock(log.mu);
  for (int p = 0; p < kPhases; ++p) {
    for (auto& e : log.ev[p]) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    log.ev[p].clear();
    log.units[p].clear();
  }
  log.on = enable != 0;
}
int goom_chain_ts_phase_stats(int phase, int64_t* launches, double* total_ms, int64_t* units) {
  if (phase < 0 || phase >= kPhases) return fail(GOOM_EINVAL, "phase must be 0..3");
  PhaseLog& log = phase_log();
  std::lock_guard<std::mutex> lock(log.mu);
  double ms = 0.0;
  int64_t prod = 0;
  for (size_t i = 0; i < log.ev[phase].size(); ++i) {
    float t = 0.0f;
    if (cudaEventSynchronize(log.ev[phase][i].second) != cudaSuccess ||
        cudaEventElapsedTime(&t, log.ev[phase][i].first, log.ev[phase][i].second) != cudaSuccess)
      return cuda_fail(cudaGetLastError(), "phase timing events");
    ms += t;
    prod += log.units[phase][i];
  }
  if (launches) *launches = (int64_t)log.ev[phase].size();
  if (total_ms) *total_ms = ms;
  if (units) *units = prod;
  return GOOM_OK;
}
int goom_chain_ts_phase3_stats(int64_t* launches, double* total_ms, int64_t* products) {
  return goom_chain_ts_phase_stats(3, launches, total_ms, products);
}

size_t goom_chain_ts_workspace_size(int64_t T, int d, int block) {
  if (T < 1 || d < 256 || d % 256 || block < 1) return 0;
  return chain_ts_workspace_bytes(T, d, block, true);
}

int goom_chain_ts(const float* U, const float* q, const uint32_t* G, int64_t T, int d, int block,
                  const float* cU, const float* cq, const uint32_t* cG, goom_c64* out,
                  float* digests4, float* oU, float* oq, uint32_t* oG, void* ws, size_t ws_bytes,
                  void* stream) {
  if (T < 1 || block < 1) return fail(GOOM_EINVAL, "T and block must be >= 1");
  if (d < 256 || d % 256) return fail(GOOM_EUNSUPPORTED, "tile-scaled chain needs d % 256 == 0");
  if (!U || !q || !G || !ws) return fail(GOOM_EINVAL, "null pointer");
  const TsBuf A = ts_of(const_cast<float*>(U), const_cast<float*>(q), const_cast<uint32_t*>(G), d);
  TsBuf ci = ts_of(const_cast<float*>(cU), const_cast<float*>(cq), const_cast<uint32_t*>(cG), d);
  TsBuf co = ts_of(oU, oq, oG, d);
  return chain_scan_ts(A, T, d, block, cU ? &ci : nullptr, reinterpret_cast<float2*>(out),
                       reinterpret_cast<float4*>(digests4), oU ? &co : nullptr,
                       reinterpret_cast<char*>(ws), ws_bytes, as_stream(stream),
                       /*tree_carries=*/true);
}

int goom_chain_ts_local(const float* U, const float* q, const uint32_t* G, int64_t T, int d,
                        int block, float* oU, float* oq, uint32_t* oG, void* ws, size_t ws_bytes,
                        void* stream) {
  if (T < 1 || block < 1) return fail(GOOM_EINVAL, "T and block must be >= 1");
  if (d < 256 || d % 256) return fail(GOOM_EUNSUPPORTED, "tile-scaled chain needs d % 256 == 0");
  if (!U || !q || !G || !ws) return fail(GOOM_EINVAL, "null pointer");
  const TsBuf A = ts_of(const_cast<float*>(U), const_cast<float*>(q), const_cast<uint32_t*>(G), d);
  cudaStream_t st = as_stream(stream);
  GOOM_TRY(chain_local(A, T, d, block, nullptr, reinterpret_cast<char*>(ws), ws_bytes, st, true));
  if (oU) {
    ChainWs w;
    GOOM_TRY(chain_ws(T, d, block, reinterpret_cast<char*>(ws), ws_bytes, w));
    TsBuf total = ts_of(oU, oq, oG, d);
    GOOM_TRY(copy_ts(total, 0, w.Cx, w.nb, 1, 1, st));
  }
  return GOOM_OK;
}

int goom_chain_ts_finish(int64_t T, int d, int block, const float* cU, const float* cq,
                         const uint32_t* cG, goom_c64* out, float* digests4, float* oU, float* oq,
                         uint32_t* oG, void* ws, size_t ws_bytes, void* stream) {
  if (T < 1 || block < 1) return fail(GOOM_EINVAL, "T and block must be >= 1");
  if (d < 256 || d % 256) return fail(GOOM_EUNSUPPORTED, "tile-scaled chain needs d % 256 == 0");
  if (!ws) return fail(GOOM_EINVAL, "null workspace");
  TsBuf ci = ts_of(const_cast<float*>(cU), const_cast<float*>(cq), const_cast<uint32_t*>(cG), d);
  TsBuf co = ts_of(oU, oq, oG, d);
  return chain_finish(T, d, block, cU ? &ci : nullptr, reinterpret_cast<float2*>(out),
                      reinterpret_cast<float4*>(digests4), oU ? &co : nullptr,
                      reinterpret_cast<char*>(ws), ws_bytes, as_stream(stream));
}

// Prefixes P_t = L_t (x) Cx[t / s] of a window that goom_chain_ts / goom_chain_ts_finish has
// just scanned with this workspace (L and the final block carries stay in it), for the
// window-local indices idx[0..n) (host array), as complex64 into out[i] and / or tile-scaled
// into (oU, oq, oG)[i]: the harness's snapshots (SURVEY §8c(5) re-anchored checks) without
// materialising the window. The tile-scaled form keeps the engine's own precision (fp32 U,
// log scale q): a complex64 log at |log| ~ 1e6 is quantised to 0.125 nats.
int goom_chain_ts_snapshots(int64_t T, int d, int block, const int64_t* idx, int n,
                            goom_c64* out, float* oU, float* oq, uint32_t* oG, void* ws,
                            size_t ws_bytes, void* stream) {
  if (T < 1 || block < 1 || n < 0) return fail(GOOM_EINVAL, "T, block >= 1 and n >= 0");
  if (d < 256 || d % 256) return fail(GOOM_EUNSUPPORTED, "tile-scaled chain needs d % 256 == 0");
  if (n == 0) return GOOM_OK;
  if (!idx || !ws || (!out && !(oU && oq && oG))) return fail(GOOM_EINVAL, "null pointer");
  ChainWs w;
  GOOM_TRY(chain_ws(T, d, block, reinterpret_cast<char*>(ws), ws_bytes, w));
  cudaStream_t st = as_stream(stream);
  const int nJ = d / 256;
  TsBuf tso;
  if (oU) {
    tso.U = oU;
    tso.q = oq;
    tso.G = oG;
    tso.d = d;
    tso.nJ = nJ;
    if (cudaMemsetAsync(oG, 0, sizeof(uint32_t) * (size_t)n * nJ, st) != cudaSuccess)
      return cuda_fail(cudaGetLastError(), "snapshot G reset");
  }
  for (int i = 0; i < n; ++i) {
    const int64_t t = idx[i];
    if (t < 0 || t >= T) return fail(GOOM_EINVAL, "snapshot index outside the window");
    if (out)
      GOOM_TRY(lmme_ts_call(w.L.in(t, 0), w.Cx.in(t / w.s, 0), kTsOutGoom,
                            reinterpret_cast<float2*>(out) + (int64_t)i * d * d, (int64_t)d * d,
                            TsOut{}, nullptr, 1, d, st));
    if (oU)
      GOOM_TRY(lmme_ts_call(w.L.in(t, 0), w.Cx.in(t / w.s, 0), kTsOutTs, nullptr, 0, tso.out(i, 0),
                            nullptr, 1, d, st));
  }
  return GOOM_OK;
}

// The block carries Cx[k] (k = kidx[i], host array of n; 0 <= k < number of blocks) of the
// window just scanned with this workspace, tile-scaled into (oU, oq, oG)[i]: the matrix the
// engine applies on the right of every local product of block k, i.e. its own P_{k s - 1}
// (the window's carry-in for k = 0). Re-anchored checks start the oracle from it.
int goom_chain_ts_carries(int64_t T, int d, int block, const int64_t* kidx, int n, float* oU,
                          float* oq, uint32_t* oG, void* ws, size_t ws_bytes, void* stream) {
  if (T < 1 || block < 1 || n < 0) return fail(GOOM_EINVAL, "T, block >= 1 and n >= 0");
  if (d < 256 || d % 256) return fail(GOOM_EUNSUPPORTED, "tile-scaled chain needs d % 256 == 0");
  if (n == 0) return GOOM_OK;
  if (!kidx || !ws || !oU || !oq || !oG) return fail(GOOM_EINVAL, "null pointer");
  ChainWs w;
  GOOM_TRY(chain_ws(T, d, block, reinterpret_cast<char*>(ws), ws_bytes, w));
  TsBuf dst;
  dst.U = oU;
  dst.q = oq;
  dst.G = oG;
  dst.d = d;
  dst.nJ = d / 256;
  for (int i = 0; i < n; ++i) {
    if (kidx[i] < 0 || kidx[i] >= w.nb) return fail(GOOM_EINVAL, "block index outside the window");
    GOOM_TRY(copy_ts(dst, i, w.Cx, kidx[i], 1, 1, as_stream(stream)));
  }
  return GOOM_OK;
}

int goom_ts_from_c64(const goom_c64* X, int64_t batch, int rows, int cols, float* U, float* q,
                     uint32_t* G, void* stream) {
  if (batch < 0 || rows < 1 || cols < 256 || cols % 256)
    return fail(GOOM_EUNSUPPORTED, "tile-scaled format needs cols % 256 == 0");
  if (batch == 0) return GOOM_OK;
  const int nJ = cols / 256;
  cudaStream_t st = as_stream(stream);
  if (cudaMemsetAsync(G, 0, sizeof(uint32_t) * (size_t)batch * nJ, st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "G reset");
  return launch_goom_to_ts(reinterpret_cast<const float2*>(X), (int64_t)rows * cols,
                           TsOut{U, q, G, (int64_t)rows * cols, (int64_t)rows * nJ, nJ}, batch,
                           rows, cols, st);
}

int goom_ts_to_c64(const float* U, const float* q, int64_t batch, int rows, int cols, goom_c64* X,
                   void* stream) {
  if (batch < 0 || rows < 1 || cols < 256 || cols % 256)
    return fail(GOOM_EUNSUPPORTED, "tile-scaled format needs cols % 256 == 0");
  if (batch == 0) return GOOM_OK;
  const int nJ = cols / 256;
  return launch_ts_to_goom(TsIn{U, q, nullptr, (int64_t)rows * cols, (int64_t)rows * nJ, nJ, 1},
                           reinterpret_cast<float2*>(X), (int64_t)rows * cols, batch, rows, cols,
                           as_stream(stream));
}

// C[b] = A(b) (x) B(b) on tile-scaled operands (matrix index b / div, stride 0 broadcasts);
// kind 0: complex64 C; 1: tile-scaled (oU, oq, oG zero-filled by the caller); 2: digests4
int goom_lmme_ts(const float* aU, const float* aq, const uint32_t* aG, int64_t a_stride,
                 int64_t a_div, const float* bU, const float* bq, const uint32_t* bG,
                 int64_t b_stride, int64_t b_div, int kind, goom_c64* C, float* oU, float* oq,
                 uint32_t* oG, float* digests4, float* parts_ws, int64_t batch, int n, int k,
                 int m, void* stream) {
  if (batch < 0) return fail(GOOM_EINVAL, "batch must be >= 0");
  if (!lmme_ts_eligible(n, k, m)) return fail(GOOM_EUNSUPPORTED, "lmme_ts needs n, k, m % 256");
  if (batch == 0) return GOOM_OK;
  const int64_t am = a_stride ? 1 : 0, bm = b_stride ? 1 : 0;
  TsProblem p{};
  p.A = TsIn{aU, aq, aG, am * (int64_t)n * k, am * (int64_t)n * (k / 256), am * (k / 256),
             a_div < 1 ? 1 : a_div};
  p.B = TsIn{bU, bq, bG, bm * (int64_t)k * m, bm * (int64_t)k * (m / 256), bm * (m / 256),
             b_div < 1 ? 1 : b_div};
  p.kind = kind;
  p.C = reinterpret_cast<float2*>(C);
  p.strideC = (int64_t)n * m;
  p.T = TsOut{oU, oq, oG, (int64_t)n * m, (int64_t)n * (m / 256), m / 256};
  p.parts = reinterpret_cast<float4*>(parts_ws);
  p.batch = batch;
  p.n = n;
  p.k = k;
  p.m = m;
  GOOM_TRY(lmme_ts(p, as_stream(stream)));
  if (kind == kTsOutDigest)
    GOOM_TRY(launch_digest_reduce(p.parts, (n / 32) * (m / 256),
                                  reinterpret_cast<float4*>(digests4), batch, as_stream(stream)));
  return GOOM_OK;
}

}  // extern "C"
