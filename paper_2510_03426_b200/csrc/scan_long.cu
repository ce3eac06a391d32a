// Long-chain scan for small matrices (d <= 32; complex64 d = 16 / 32 / 64 fold on tcgen05 at the
// leaf level, scan_long_tc.cu): reduce-then-scan over LMME combines.
//
// The reference's two-level tree (_scan_affine_stack, scan.py:181-214) has a sequential
// depth of s + T/s combines — ~2,000 dependent LMMEs at T = 2^20 however s is chosen —
// and moves 32 d^2 bytes per element (leaves in, local products out and back, prefixes
// out). This engine computes the same prefixes P_t = A_t (x) ... (x) A_0 (x) carry_in
// with a different but fixed tree, for chains far longer than any block:
//   R-pass  tot[k]  = A_{ks+s-1} (x) ... (x) A_{ks}            (reads the leaves)
//   scan    incl[k] = tot[k] (x) ... (x) tot[0] (x) carry_in    (the same engine, recursively)
//   S-pass  P_t     = A_t (x) P_{t-1}, P_{ks-1} = incl[k-1]     (reads the leaves again,
//                                                               writes every prefix)
// 24 d^2 bytes per element (complex64: 8 d^2 per pass over the leaves, 8 d^2 out), two
// LMMEs per element, and a sequential depth of O(s log_s T).
//
// One chain (a block of s consecutive leaves) belongs to a group of D lanes (D = 8, 16 or
// 32 for d <= D: 4, 2 or 1 chains per warp) that synchronises only itself. Per step
// (P <- A_t (x) P), all through the group's shared memory:
//   * the leaf arrives by cp.async (8-byte, coalesced) into a padded stage one step ahead;
//   * lane i transforms leaf row i (clamped row scale a_i, sign * exp) into column i of
//     leftT; lane j transforms column j of the state (b_j, sign * exp) into right;
//   * each lane accumulates a TR x TC register tile of the product (4 x 8 at D = 32: three
//     16-byte shared loads per 32 FMAs instead of two per 8) and writes it back to the
//     state as complex GOOMs, (log|I| + a) + b;
//   * the state is copied out to HBM coalesced (S-pass: every prefix; R-pass: the total).
// Every combine is lmme_small's arithmetic (lmme_simt.cu: clamped scales (Eq. 11,
// core.py:252-255), sign * exp, one FMA per term in ascending k, (log|I| + a) + b), so
// each step is bitwise the generic LMME of the same operands and a single chain is
// bitwise the sequential fold (scan_chain with block >= T).
#include <cstdlib>

#include "goom_internal.cuh"

namespace goom {

namespace {

constexpr int kLongS0 = 64;   // chain length at the leaf level
constexpr int kLongTop = 32;  // an input this short runs as one chain (the sequential fold)

// the upper levels (chains of totals) are latency-bound: each SIMT fold step is a ~1 us
// dependent chain whatever the load, so their cost is the tree's sequential depth (2 s per
// level plus the top chain) and ~2 us per launch. Chains of s = 4 up to a top chain of 4
// measured best for the lane-group fold (d <= 32: 2-4% off the whole scan against 16 / 32);
// the d = 64 tcgen05 fold keeps 16 / 32 (s = 4 / 8 measured 1.5% / 0% slower;
// profiles/r2_long_upper_tree.txt). GOOM_LONG_S / GOOM_LONG_TOP override both for measurement.
struct UpperTree {
  int s, top;
};
inline UpperTree upper_tree(int d) {
  static const UpperTree env = [] {
    UpperTree v{0, 0};
    if (const char* e = getenv("GOOM_LONG_S")) v.s = atoi(e) >= 2 ? atoi(e) : 0;
    if (const char* e = getenv("GOOM_LONG_TOP")) v.top = atoi(e) >= 1 ? atoi(e) : 0;
    return v;
  }();
  UpperTree u = d > 32 ? UpperTree{16, 32} : UpperTree{4, 4};
  if (env.s) u.s = env.s;
  if (env.top) u.top = env.top;
  return u;
}
inline int64_t level_s(int level, int d) { return level == 0 ? kLongS0 : upper_tree(d).s; }
inline int64_t level_top(int level, int d) {
  return level == 0 ? kLongTop : upper_tree(d).top;
}

inline size_t rup(size_t x) { return (x + 255) & ~size_t(255); }

template <class R, int D>
struct LongCfg {
  static constexpr int TR = D == 8 ? 2 : 4;        // product rows per lane
  static constexpr int TC = D == 32 ? 8 : 4;       // product columns per lane
  static constexpr int NCQ = D / TC;               // column groups
  static_assert((D / TR) * NCQ == D, "tile grid must cover the group");
  static constexpr int P = D + 1;                  // complex pitch of stage / state (odd)
  static constexpr int kThreads = D == 32 ? 64 : 128;
  static constexpr int kChains = kThreads / D;     // chains per CTA
};

template <class R, int D>
struct alignas(16) LongSmem {       // one chain's staging
  R leftT[D * D];                   // transformed leaf, transposed: [k][i]
  R right[D * D];                   // transformed state: [k][j]
  R sa[D], sb[D];                   // clamped row / column scales
  Cx<R> stage[D * (D + 1)];         // the incoming leaf, padded rows
  Cx<R> st[D * (D + 1)];            // the state P, padded rows
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void lds_n(const float* p, float (&v)[N]) {
  if constexpr (N == 2) {
    const float2 x = *reinterpret_cast<const float2*>(p);
    v[0] = x.x, v[1] = x.y;
  } else {
#pragma unroll
    for (int q = 0; q < N; q += 4) {
      const float4 x = *reinterpret_cast<const float4*>(p + q);
      v[q] = x.x, v[q + 1] = x.y, v[q + 2] = x.z, v[q + 3] = x.w;
    }
  }
}
template <int N>
__device__ __forceinline__ void lds_n(const double* p, double (&v)[N]) {
#pragma unroll
  for (int q = 0; q < N; q += 2) {
    const double2 x = *reinterpret_cast<const double2*>(p + q);
    v[q] = x.x, v[q + 1] = x.y;
  }
}

// element e of a dense d x d matrix -> its slot in a padded [D][D + 1] buffer
template <int D, bool kFull>
__device__ __forceinline__ int pad_slot(int e, int d) {
  if (kFull) return e + e / D;  // row e / D, column e % D
  const int r = e / d;
  return r * (D + 1) + (e - r * d);
}

// dense (global) -> padded (shared), asynchronous: lane gl copies elements gl, gl + D, ...
template <class R, int D, bool kFull>
__device__ __forceinline__ void copy_in_async(Cx<R>* dst, const Cx<R>* __restrict__ src, int d,
                                              int gl) {
  const int n = d * d;
#pragma unroll 4
  for (int e = gl; e < n; e += D) {
    if constexpr (sizeof(R) == 4) cp_async8(dst + pad_slot<D, kFull>(e, d), src + e);
    else cp_async16(dst + pad_slot<D, kFull>(e, d), src + e);
  }
}
// (log, any phase) -> (log, 0 or pi): the state keeps canonical signs
template <class C>
__device__ __forceinline__ C canonical(C z) {
  z.y = phase_negative(z.y) ? pi_of<decltype(z.x)>() : decltype(z.x)(0);
  return z;
}
template <class R, int D, bool kFull>
__device__ __forceinline__ void copy_in(Cx<R>* dst, const Cx<R>* __restrict__ src, int d, int gl) {
  const int n = d * d;
  for (int e = gl; e < n; e += D) dst[pad_slot<D, kFull>(e, d)] = canonical(src[e]);
}
// padded (shared) -> dense (global), coalesced
template <class R, int D, bool kFull>
__device__ __forceinline__ void copy_out(Cx<R>* __restrict__ dst, const Cx<R>* src, int d, int gl) {
  const int n = d * d;
  for (int e = gl; e < n; e += D) dst[e] = src[pad_slot<D, kFull>(e, d)];
}

// chains k = 0 .. ceil(T / s) - 1 over leaves [ks, min(ks + s, T)); chain k starts from
// carry0 (k = 0) or carries[k - 1] (k >= 1) when given, else from its first leaf (raw).
// out (nullable): every state; tot (nullable): each chain's last state.
template <class R, int D, bool kFull>
__global__ void __launch_bounds__(LongCfg<R, D>::kThreads)
    long_fold_kernel(const Cx<R>* __restrict__ A, int64_t T, int d_rt, int64_t s,
                     const Cx<R>* __restrict__ carry0, const Cx<R>* __restrict__ carries,
                     Cx<R>* __restrict__ out, Cx<R>* __restrict__ tot) {
  using Cfg = LongCfg<R, D>;
  using C = Cx<R>;
  constexpr int TR = Cfg::TR, TC = Cfg::TC, P = Cfg::P;
  const int d = kFull ? D : d_rt;  // d == D: every bound and slot is a compile-time constant
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int gl = lane % D;                      // lane in the group
  const int grp = threadIdx.x / D;              // chain slot in the CTA
  const unsigned gmask = D == 32 ? 0xffffffffu : (((1u << D) - 1u) << (lane - gl));
  LongSmem<R, D>& sm = reinterpret_cast<LongSmem<R, D>*>(smem_raw)[grp];
  const int64_t chain = (int64_t)blockIdx.x * Cfg::kChains + grp;
  const int64_t t0 = chain * s;
  if (t0 >= T) return;  // group-uniform: the group's syncs only name its own lanes
  const int64_t t1 = t0 + s < T ? t0 + s : T;
  const int64_t mat = (int64_t)d * d;
  const int i0 = (gl / Cfg::NCQ) * TR, j0 = (gl % Cfg::NCQ) * TC;

  copy_in_async<R, D, kFull>(sm.stage, A + t0 * mat, d, gl);
  cp_async_commit();
  const C* cin = chain == 0 ? carry0 : (carries ? carries + (chain - 1) * mat : nullptr);
  bool has = cin != nullptr;
  if (has) copy_in<R, D, kFull>(sm.st, cin, d, gl);
  cp_async_wait_all();
  __syncwarp(gmask);
  for (int64_t t = t0; t < t1; ++t) {
    const bool more = t + 1 < t1;
    const bool first = !has;  // this step only copies the leaf in as the state
    if (first) {  // the chain's first leaf is its first state (output raw, like the tree's L[ks])
      if (out) copy_out<R, D, kFull>(out + t * mat, sm.stage, d, gl);
#pragma unroll 4
      for (int j = 0; j < D; ++j) sm.st[gl * P + j] = canonical(sm.stage[gl * P + j]);
      __syncwarp(gmask);
      if (more) copy_in_async<R, D, kFull>(sm.stage, A + (t + 1) * mat, d, gl);
      cp_async_commit();
    } else {
      // left operand row gl: a = max(rowmax, 0), sign * exp(x - a) into column gl of leftT
      {
        R ai = R(-INFINITY);
#pragma unroll 8
        for (int k = 0; k < D; ++k)
          if (k < d) ai = gmax(ai, sm.stage[gl * P + k].x);
        ai = gmax(ai, R(0));
#pragma unroll 8
        for (int k = 0; k < D; ++k) {
          R v = R(0);
          if (k < d && gl < d) {
            const C z = sm.stage[gl * P + k];
            v = goom_sign_t<R>(z.y) * gexp(z.x - ai);
          }
          sm.leftT[k * D + gl] = v;
        }
        sm.sa[gl] = ai;
      }
      // right operand column gl: b = max(colmax, 0), sign * exp(x - b) into right
      {
        R bj = R(-INFINITY);
#pragma unroll 8
        for (int k = 0; k < D; ++k)
          if (k < d) bj = gmax(bj, sm.st[k * P + gl].x);
        bj = gmax(bj, R(0));
#pragma unroll 8
        for (int k = 0; k < D; ++k) {
          R v = R(0);
          if (k < d && gl < d) {
            const C z = sm.st[k * P + gl];  // canonical: the phase is exactly 0 or pi
            v = (z.y != R(0) ? R(-1) : R(1)) * gexp(z.x - bj);
          }
          sm.right[k * D + gl] = v;
        }
        sm.sb[gl] = bj;
      }
      __syncwarp(gmask);
      if (more) copy_in_async<R, D, kFull>(sm.stage, A + (t + 1) * mat, d, gl);  // stage is free
      cp_async_commit();
      // TR x TC tile of the product, one FMA per term in ascending k
      R acc[TR][TC];
#pragma unroll
      for (int r = 0; r < TR; ++r)
#pragma unroll
        for (int c = 0; c < TC; ++c) acc[r][c] = R(0);
#pragma unroll 4
      for (int k = 0; k < D; ++k) {
        if (k < d) {
          R lv[TR], rv[TC];
          lds_n<TR>(&sm.leftT[k * D + i0], lv);
          lds_n<TC>(&sm.right[k * D + j0], rv);
#pragma unroll
          for (int r = 0; r < TR; ++r)
#pragma unroll
            for (int c = 0; c < TC; ++c) acc[r][c] = gfma(lv[r], rv[c], acc[r][c]);
        }
      }
      // epilogue into the state (its last readers passed the sync above)
      R bv[TC];
      lds_n<TC>(&sm.sb[j0], bv);
#pragma unroll
      for (int r = 0; r < TR; ++r) {
        const R a = sm.sa[i0 + r];
#pragma unroll
        for (int c = 0; c < TC; ++c) sm.st[(i0 + r) * P + j0 + c] = lmme_out<R>(acc[r][c], a, bv[c]);
      }
    }
    cp_async_wait_all();
    __syncwarp(gmask);  // the state and the next leaf are complete
    if (out && !first) copy_out<R, D, kFull>(out + t * mat, sm.st, d, gl);
    has = true;
  }
  if (tot) copy_out<R, D, kFull>(tot + chain * mat, sm.st, d, gl);
}

template <class R, int D>
int launch_fold_d(const Cx<R>* A, int64_t T, int d, int64_t s, const Cx<R>* carry0,
                  const Cx<R>* carries, Cx<R>* out, Cx<R>* tot, cudaStream_t st) {
  using Cfg = LongCfg<R, D>;
  const int bytes = Cfg::kChains * (int)sizeof(LongSmem<R, D>);
  auto kern = d == D ? long_fold_kernel<R, D, true> : long_fold_kernel<R, D, false>;
  if (bytes > 48 * 1024) GOOM_TRY(smem_attr((const void*)kern, bytes, "long_fold smem"));
  const int64_t chains = (T + s - 1) / s;
  const int64_t grid = (chains + Cfg::kChains - 1) / Cfg::kChains;
  kern<<<(unsigned)grid, Cfg::kThreads, bytes, st>>>(A, T, d, s, carry0, carries, out, tot);
  GOOM_CHECK_LAUNCH("long_fold_kernel");
  return GOOM_OK;
}

template <class R>
int launch_fold(const Cx<R>* A, int64_t T, int d, int64_t s, const Cx<R>* carry0,
                const Cx<R>* carries, Cx<R>* out, Cx<R>* tot, cudaStream_t st) {
  if constexpr (sizeof(R) == 4) {
    // complex64 d = 64, and d = 16 / 32 at the leaf level (chains of kLongS0): the
    // tile-resident tcgen05 fold (scan_long_tc.cu); the short upper levels (and every level
    // with GOOM_LONG_TC=0) keep the lane-group fold below
    static const bool tc_small = [] {
      const char* e = getenv("GOOM_LONG_TC");
      return !(e && atoi(e) == 0);
    }();
    if (fold_tc_eligible(d) && (d == 64 || (tc_small && s >= kLongS0)))
      return launch_fold_tc(A, T, d, s, carry0, carries, out, tot, st);
  }
  if (d <= 8) return launch_fold_d<R, 8>(A, T, d, s, carry0, carries, out, tot, st);
  if (d <= 16) return launch_fold_d<R, 16>(A, T, d, s, carry0, carries, out, tot, st);
  return launch_fold_d<R, 32>(A, T, d, s, carry0, carries, out, tot, st);
}

template <class R>
int long_scan(const Cx<R>* A, Cx<R>* out, int64_t T, int d, const Cx<R>* carry_in, char* ws,
              cudaStream_t st, int level) {
  if (T <= level_top(level, d))
    return launch_fold<R>(A, T, d, T, carry_in, nullptr, out, nullptr, st);
  const int64_t s = level_s(level, d);
  const int64_t nb = (T + s - 1) / s;
  const size_t mats = rup(sizeof(Cx<R>) * (size_t)nb * d * d);
  Cx<R>* tot = reinterpret_cast<Cx<R>*>(ws);
  Cx<R>* incl = reinterpret_cast<Cx<R>*>(ws + mats);
  GOOM_TRY(launch_fold<R>(A, T, d, s, nullptr, nullptr, nullptr, tot, st));        // R-pass
  GOOM_TRY(long_scan<R>(tot, incl, nb, d, carry_in, ws + 2 * mats, st, level + 1));  // totals
  return launch_fold<R>(A, T, d, s, carry_in, incl, out, nullptr, st);             // S-pass
}

}  // namespace

template <class R>
bool chain_long_eligible(int d) { return (d >= 1 && d <= 32) || (sizeof(R) == 4 && d == 64); }

template <class R>
size_t chain_long_workspace_bytes(int64_t T, int d) {
  size_t total = 256;
  int64_t n = T;
  for (int level = 0; n > level_top(level, d); ++level) {
    const int64_t s = level_s(level, d);
    const int64_t nb = (n + s - 1) / s;
    total += 2 * rup(sizeof(Cx<R>) * (size_t)nb * d * d);
    n = nb;
  }
  return total;
}

template <class R>
int chain_scan_long(const Cx<R>* A, Cx<R>* out, int64_t T, int d, const Cx<R>* carry_in,
                    void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!chain_long_eligible<R>(d))
    return fail(GOOM_EUNSUPPORTED, "long-chain scan needs d <= 32 (or d = 64, complex64)");
  if (ws_bytes < chain_long_workspace_bytes<R>(T, d) || !ws)
    return fail(GOOM_EWORKSPACE, "long-chain scan workspace too small");
  return long_scan<R>(A, out, T, d, carry_in, reinterpret_cast<char*>(ws), st, 0);
}

template bool chain_long_eligible<float>(int);
template bool chain_long_eligible<double>(int);
template size_t chain_long_workspace_bytes<float>(int64_t, int);
template size_t chain_long_workspace_bytes<double>(int64_t, int);
template int chain_scan_long<float>(const float2*, float2*, int64_t, int, const float2*, void*,
                                    size_t, cudaStream_t);
template int chain_scan_long<double>(const double2*, double2*, int64_t, int, const double2*, void*,
                                     size_t, cudaStream_t);

}  // namespace goom

using namespace goom;

namespace {
template <class R>
int long_entry(const void* A, void* out, int64_t T, int d, const void* carry_in, void* ws,
               size_t ws_bytes, void* stream) {
  if (T < 1) return fail(GOOM_EINVAL, "T must be >= 1");
  if (d < 1) return fail(GOOM_ESHAPE, "d must be >= 1");
  if (!A || !out) return fail(GOOM_EINVAL, "null pointer");
  return chain_scan_long<R>(reinterpret_cast<const Cx<R>*>(A), reinterpret_cast<Cx<R>*>(out), T,
                            d, reinterpret_cast<const Cx<R>*>(carry_in), ws, ws_bytes,
                            as_stream(stream));
}
}  // namespace

extern "C" {

size_t goom_scan_chain_long_workspace_size(int64_t T, int d) {
  if (T < 1 || !chain_long_eligible<float>(d)) return 0;
  return chain_long_workspace_bytes<float>(T, d);
}
size_t goom_scan_chain_long_workspace_size_c128(int64_t T, int d) {
  if (T < 1 || !chain_long_eligible<double>(d)) return 0;
  return chain_long_workspace_bytes<double>(T, d);
}
int goom_scan_chain_long_c64(const goom_c64* A, goom_c64* out, int64_t T, int d,
                             const goom_c64* carry_in, void* ws, size_t ws_bytes, void* stream) {
  return long_entry<float>(A, out, T, d, carry_in, ws, ws_bytes, stream);
}
int goom_scan_chain_long_c128(const goom_c128* A, goom_c128* out, int64_t T, int d,
                              const goom_c128* carry_in, void* ws, size_t ws_bytes, void* stream) {
  return long_entry<double>(A, out, T, d, carry_in, ws, ws_bytes, stream);
}

}  // extern "C"
