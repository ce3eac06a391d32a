// Selective-reset product-chain scan (scan.py:342-504 + lyapunov.py:146-278).
//
// Structure (the reference's strided walk, scan.py:356-428, on the device):
//   1. local products per tile of s = check_interval leaves, batched across
//      tiles (the chain engine's phase 1; with consume_leaf also the variant
//      whose tile starts at the identity, scan.py:317-339);
//   2. ONE persistent CTA walks the tiles in order. Per tile it forms the tile
//      total el = loc[p] (x) carry with a CTA-level LMME (carry resident in
//      shared memory), evaluates the policy predicate on el in FP64, and on a
//      fire replaces the carry by the policy's reset value and records the
//      site p+1. The predicate and the reset are fused into the walk — no host
//      round trip per tile;
//   3. every position is materialised in one batched LMME, loc[t] (x) carry[t/s].
// check_interval == 1 is the same machinery with s = 1 (every position tested):
// the per-position walk of scan.py:431-484 collapses to the sequential fold,
// whose reset sites the reference proves identical (scan.py:9-12).
//
// Policies (FP64 inside the CTA, d <= 64):
//   colinearity: log-unit-normalised columns (lyapunov.py:255-263); fire on an
//     all-zero column, on max_{i<j} |G_ij| > threshold (G = R^T R) or on
//     log|det R| < log(volume_floor) / det == 0 (LU with partial pivoting, as
//     LAPACK getrf behind np.linalg.slogdet);
//     reset = the CGS2 orthonormal basis (lyapunov.py:175-219). It is computed
//     as Householder QR with column signs chosen so diag(R) > 0 — the same Q
//     (QR with positive diagonal is unique), rank-deficiency at |R_jj| < 64 eps.
//   norm-threshold: fire when max_j log||col_j|| > threshold; reset = LAPACK-
//     convention Householder Q of the unit-column matrix (np.linalg.qr,
//     pkg/tests/test_scan.py:60-75).
#include <vector>

#include <cstdio>
#include <cstdlib>

#include "goom_internal.cuh"
#include "tc_ptx.cuh"

namespace goom {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxD = 64;

// Walk phase clocks (thread 0 of the single walk CTA), read back by the host when
// GOOM_WALK_TIMING is set: [0] tile LMME / copy, [1] carry store, [2] column norms,
// [3] Gram, [4] LU volume test, [5] reset (norms + QR + Q), [6] reset log export,
// [7] carry copy, [8] tiles, [9] fires.
__device__ unsigned long long g_walk_prof[16];
__device__ __forceinline__ void prof_add(bool on, int slot, long long& t0) {
  if (on && threadIdx.x == 0) {
    const long long t = clock64();
    g_walk_prof[slot] += (unsigned long long)(t - t0);
    t0 = t;
  }
}

struct Policy {
  int kind;
  int interval;
  int consume;
  double threshold;
  double log_floor;
  int timing;
};

// Shared-memory carve-up of the walk CTA; Rt is the chain's backing precision.
template <class Rt>
struct Smem {
  Cx<Rt>* carry;  // d*d
  Cx<Rt>* el;     // d*d
  double* R;      // d*d  (R and W also host the LMME operand planes tl / tr)
  double* W;      // d*d
  Rt* tl;         // d*d (aliases R)
  Rt* tr;         // d*d
  Rt* scal;       // 2d
  double* vec;    // 2d
  double* red;    // 2 * kWarps
  double* part;   // 4 * kMaxD: per-(row chunk, column) partials of the column-parallel kernels
  uint64_t* mbar;  // 1: the walk's operand prefetch barrier
  int* ints;      // 8
};

template <class Rt>
inline size_t smem_bytes(int d) {
  size_t dd = (size_t)d * d;
  return 2 * dd * sizeof(Cx<Rt>) + 2 * dd * sizeof(double) + 2 * d * sizeof(Rt) +
         2 * d * sizeof(double) + 2 * kWarps * sizeof(double) + 4 * kMaxD * sizeof(double) +
         16 + 16 * sizeof(int) + 64;
}

template <class Rt>
__device__ Smem<Rt> carve(char* base, int d) {
  Smem<Rt> s;
  size_t dd = (size_t)d * d;
  s.carry = reinterpret_cast<Cx<Rt>*>(base);
  s.el = s.carry + dd;
  s.R = reinterpret_cast<double*>(s.el + dd);
  s.W = s.R + dd;
  s.tl = reinterpret_cast<Rt*>(s.R);
  s.tr = s.tl + dd;
  s.vec = s.W + dd;
  s.red = s.vec + 2 * d;
  s.part = s.red + 2 * kWarps;
  s.mbar = reinterpret_cast<uint64_t*>(s.part + 4 * kMaxD);
  s.scal = reinterpret_cast<Rt*>(s.mbar + 2);
  s.ints = reinterpret_cast<int*>(s.scal + 2 * d);
  return s;
}

__device__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double r = red[0];
  for (int i = 1; i < kWarps; ++i) r = fmax(r, red[i]);
  return r;
}

// Eq. 10-12 at the chain's precision in one CTA, split so that the left operand's half
// (clamped row maxima, scaled exponentials) can be produced ahead of time:
//   lmme_left   sm.scal[0, d) = max(row max of Lg, 0); sm.tl[k d + i] = s e^{Lg_ik - scal_i}
//   lmme_right  out (smem) = (tl) (x) Rs with Rs's clamped column maxima, the GEMM and
//               the log / max-add-back epilogue
// Same per-output FMA order as the SIMT kernels (bitwise-identical products).
template <class Rt>
__device__ void lmme_left(const Cx<Rt>* __restrict__ Lg, int d, Rt* scal, Rt* tl,
                          const Smem<Rt>& sm) {
  const int tid = threadIdx.x, cc = tid & (kMaxD - 1), ch = tid / kMaxD;
  Rt mr = Rt(-INFINITY);
  if (cc < d)
    for (int t = ch; t < d; t += 4) mr = gmax(mr, Lg[cc * d + t].x);
  sm.part[ch * kMaxD + cc] = (double)mr;
  __syncthreads();
  if (cc < d && ch == 0)
    scal[cc] = gmax(gmax(gmax((Rt)sm.part[cc], (Rt)sm.part[kMaxD + cc]),
                         gmax((Rt)sm.part[2 * kMaxD + cc], (Rt)sm.part[3 * kMaxD + cc])),
                    Rt(0));
  __syncthreads();
  for (int e = tid; e < d * d; e += kThreads) {
    const int i = e / d, j = e % d;
    const Cx<Rt> z = Lg[e];  // row i, column j (= k index)
    tl[j * d + i] = goom_sign_t<Rt>(z.y) * gexp(z.x - scal[i]);
  }
  __syncthreads();
}

template <class Rt>
__device__ void lmme_right(const Cx<Rt>* Rs, Cx<Rt>* out, int d, const Smem<Rt>& sm,
                           bool tm = false) {
  const int tid = threadIdx.x, cc = tid & (kMaxD - 1), ch = tid / kMaxD;
  long long t0 = clock64();
  Rt mc = Rt(-INFINITY);
  if (cc < d)
    for (int t = ch; t < d; t += 4) mc = gmax(mc, Rs[t * d + cc].x);
  sm.part[ch * kMaxD + cc] = (double)mc;
  __syncthreads();
  if (cc < d && ch == 0)
    sm.scal[d + cc] = gmax(gmax(gmax((Rt)sm.part[cc], (Rt)sm.part[kMaxD + cc]),
                                gmax((Rt)sm.part[2 * kMaxD + cc], (Rt)sm.part[3 * kMaxD + cc])),
                           Rt(0));
  __syncthreads();
  for (int e = tid; e < d * d; e += kThreads) {
    const Cx<Rt> q = Rs[e];  // row (= k index), column j
    sm.tr[e] = goom_sign_t<Rt>(q.y) * gexp(q.x - sm.scal[d + e % d]);
  }
  __syncthreads();
  prof_add(tm, 10, t0);
  const int ty = tid >> 4, tx = tid & 15;
  Rt acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = Rt(0);
  for (int kk = 0; kk < d; ++kk) {
    Rt av[4], bv[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int i = ty + 16 * r;
      av[r] = i < d ? sm.tl[kk * d + i] : Rt(0);
      int j = tx + 16 * r;
      bv[r] = j < d ? sm.tr[kk * d + j] : Rt(0);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = gfma(av[r], bv[c], acc[r][c]);
  }
  if (tm) __syncthreads();
  prof_add(tm, 11, t0);
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    int i = ty + 16 * r;
    if (i >= d) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      int j = tx + 16 * c;
      if (j >= d) continue;
      out[i * d + j] = lmme_out<Rt>(acc[r][c], sm.scal[i], sm.scal[d + j]);
    }
  }
  __syncthreads();
  prof_add(tm, 12, t0);
}

// out (smem) = Lg (global) (x) Rs (smem)
template <class Rt>
__device__ void block_lmme(const Cx<Rt>* __restrict__ Lg, const Cx<Rt>* Rs, Cx<Rt>* out, int d,
                           const Smem<Rt>& sm) {
  lmme_left(Lg, d, sm.scal, sm.tl, sm);
  lmme_right(Rs, out, d, sm);
}

// The walk's left operands ahead of time, batched over tiles: CTA k writes tile k's
// (position min(k s + s, T) - 1 of loc) clamped row maxima to rs[k d ..] and its scaled
// exponentials, in the walk's sm.tl layout, to P[k d^2 ..] — the walk then streams
// them into shared memory with one bulk copy instead of reading and exponentiating the
// GOOM matrix on its sequential path.
template <class Rt>
__global__ void __launch_bounds__(kThreads, 1)
    tile_operand_kernel(const Cx<Rt>* __restrict__ loc, int64_t T, int d, int s,
                        Rt* __restrict__ P, Rt* __restrict__ rs) {
  extern __shared__ __align__(16) char smem_raw[];
  Smem<Rt> sm = carve<Rt>(smem_raw, d);
  const int64_t dd = (int64_t)d * d;
  const int64_t lo = (int64_t)blockIdx.x * s;
  const int64_t p = (lo + s < T ? lo + s : T) - 1;
  lmme_left(loc + p * dd, d, sm.scal, sm.tl, sm);
  for (int64_t e = threadIdx.x; e < dd; e += kThreads) P[blockIdx.x * dd + e] = sm.tl[e];
  for (int i = threadIdx.x; i < d; i += kThreads) rs[blockIdx.x * d + i] = sm.scal[i];
}

// ---- register-resident column kernels (d <= 64, 256 threads) -------------------------
// Warp w owns columns 8w .. 8w+7; lane l holds column c = 8w + l/4, rows r = l%4 + 4i
// (i < 16) in registers. Column reductions are 4-lane shuffles, so the column norms, the
// Householder updates and the Q accumulation need no CTA barrier; the QR's only barrier
// per column publishes the reflector.
struct ColLane {
  int c, rc;
};
__device__ __forceinline__ ColLane col_lane() {
  return ColLane{(int)(threadIdx.x >> 5) * 8 + (int)((threadIdx.x & 31) >> 2), (int)(threadIdx.x & 3)};
}
__device__ __forceinline__ double quad_sum(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v + __shfl_xor_sync(0xffffffffu, v, 2);
}
__device__ __forceinline__ double quad_max(double v) {
  v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fmax(v, __shfl_xor_sync(0xffffffffu, v, 2));
}

__device__ __forceinline__ double tree_sum16(double (&a)[16]) {
#pragma unroll
  for (int w = 8; w > 0; w >>= 1)
#pragma unroll
    for (int i = 0; i < w; ++i) a[i] += a[i + w];
  return a[0];
}

// Log-unit-normalised columns (lyapunov.py:255-263) of X (smem GOOMs, d x d): this
// thread's column into x, the whole matrix into sm.R (row-major, for the Gram) and the
// column log-norms nu_c = m + 1/2 log sum e^{2(L - m)} into sm.vec[0, d). Returns true
// (CTA-uniform) when some column is all zero.
template <class Rt, bool kStoreR = true>
__device__ bool unit_columns_regs(const Cx<Rt>* X, int d, double (&x)[16], const Smem<Rt>& sm) {
  const ColLane L = col_lane();
  const bool live = L.c < d;
  double lg[16];
  double m = -INFINITY;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int r = L.rc + 4 * i;
    lg[i] = -INFINITY;
    x[i] = 1.0;
    if (live && r < d) {
      const Cx<Rt> z = X[r * d + L.c];
      lg[i] = (double)z.x;
      x[i] = (double)goom_sign_t<Rt>(z.y);
    }
    m = fmax(m, lg[i]);
  }
  m = quad_max(m);
  const bool zero = live && m == -INFINITY;
  double s0 = 0.0, s1 = 0.0;
  if (m != -INFINITY) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      s0 += exp(2.0 * (lg[i] - m));
      s1 += exp(2.0 * (lg[i + 1] - m));
    }
  }
  const double ss = quad_sum(s0 + s1);  // every lane: full-warp shuffle
  const double nu = m == -INFINITY ? -INFINITY : m + 0.5 * log(ss);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int r = L.rc + 4 * i;
    x[i] = (live && r < d && !zero) ? x[i] * exp(lg[i] - nu) : 0.0;
    if (kStoreR && live && r < d) sm.R[r * d + L.c] = x[i];
  }
  if (live && L.rc == 0) sm.vec[L.c] = nu;
  return __syncthreads_or(zero) != 0;
}

// max_{i<j} |G_ij|, G = R^T R of sm.R (the unit-column Gram, lyapunov.py:146-155):
// 4 x 4 register tiles, one pass over the rows.
template <class Rt>
__device__ double gram_offdiag_max(int d, const Smem<Rt>& sm) {
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int r = 0; r < d; ++r) {
    double av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = ty + 16 * a, j = tx + 16 * a;
      av[a] = i < d ? sm.R[r * d + i] : 0.0;
      bv[a] = j < d ? sm.R[r * d + j] : 0.0;
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
  }
  double g = 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ty + 16 * a, j = tx + 16 * b;
      if (i < j && j < d) g = fmax(g, fabs(acc[a][b]));
    }
  return block_max(g, sm.red);
}

// Householder QR (LAPACK dgeqr2 / dlarfg arithmetic) of the register-resident matrix.
// Reflector j goes to sm.W as row j of V^T (v_j[j] = 1, zero above), tau_j to
// sm.vec[0, d), R_jj to sm.vec[d, 2d). x is consumed. One CTA barrier per column.
template <class Rt>
__device__ void qr_regs(double (&x)[16], int d, const Smem<Rt>& sm) {
  const ColLane L = col_lane();
  const int warp = threadIdx.x >> 5, qbase = threadIdx.x & 28;
  double* Vt = sm.W;
  double* tau = sm.vec;
  double* diag = sm.vec + d;
  for (int j = 0; j < d; ++j) {
    if (warp < (j >> 3)) break;   // every column of this warp is final; the warps still
                                  // active sync on a named barrier sized to them
    if (warp == (j >> 3)) {       // the warp owning column j builds the reflector; full-warp
                                  // shuffles, only the quad of column j keeps its values
      double sq[16], alpha = 0.0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int r = L.rc + 4 * i;
        sq[i] = (r > j && r < d) ? x[i] * x[i] : 0.0;  // independent products, tree sum
        if (r == j) alpha = x[i];
      }
      const double s = quad_sum(tree_sum16(sq));
      alpha = __shfl_sync(0xffffffffu, alpha, qbase | (j & 3));
      if (L.c == j) {
        // dlarfg: beta = -sign(alpha) ||(alpha, x)||, tau = (beta - alpha) / beta,
        // v = x / (alpha - beta); one rsqrt and one reciprocal instead of sqrt + 2 divisions
        double t = 0.0, beta = alpha, scale = 0.0;
        if (s != 0.0) {
          const double n2 = fma(alpha, alpha, s);
          const double rn = rsqrt(n2);
          const double nrm = n2 * rn;
          beta = -copysign(nrm, alpha);
          t = fma(fabs(alpha), rn, 1.0);                 // (beta - alpha) / beta
          scale = copysign(__drcp_rn(fabs(alpha) + nrm), alpha);  // 1 / (alpha - beta)
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int r = L.rc + 4 * i;
          if (r < d) Vt[j * d + r] = r > j ? x[i] * scale : (r == j ? 1.0 : 0.0);
        }
        if (L.rc == 0) {
          tau[j] = t;
          diag[j] = beta;
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"((kWarps - (j >> 3)) * 32) : "memory");
    const double t = tau[j];
    if (t != 0.0) {
      double pr[16], v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int r = L.rc + 4 * i;
        v[i] = (r >= j && r < d) ? Vt[j * d + r] : 0.0;
        pr[i] = v[i] * x[i];
      }
      const double w = t * quad_sum(tree_sum16(pr));
      if (L.c > j && L.c < d) {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fma(-w, v[i], x[i]);
      }
    }
  }
  __syncthreads();
}

// Q = H_0 ... H_{d-1} I (LAPACK dorg2r order) from qr_regs' reflectors into q, this
// thread's column; no barriers (every warp applies all reflectors to its own columns).
// positive_diag flips columns so that diag(R) > 0 (the CGS2 basis, lyapunov.py:175-194).
template <class Rt>
__device__ void q_regs(double (&q)[16], int d, bool positive_diag, const Smem<Rt>& sm) {
  const ColLane L = col_lane();
  const double* Vt = sm.W;
  const double* tau = sm.vec;
#pragma unroll
  for (int i = 0; i < 16; ++i) q[i] = (L.rc + 4 * i == L.c) ? 1.0 : 0.0;
  for (int j = d - 1; j >= 0; --j) {
    const double t = tau[j];
    if (t == 0.0) continue;
    double p0 = 0.0, p1 = 0.0, v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int r = L.rc + 4 * i;
      v[i] = (r >= j && r < d) ? Vt[j * d + r] : 0.0;
      if (i & 1) p1 = fma(v[i], q[i], p1);
      else p0 = fma(v[i], q[i], p0);
    }
    const double w = t * quad_sum(p0 + p1);
#pragma unroll
    for (int i = 0; i < 16; ++i) q[i] = fma(-w, v[i], q[i]);
  }
  if (positive_diag && L.c < d && sm.vec[d + L.c] < 0.0)
#pragma unroll
    for (int i = 0; i < 16; ++i) q[i] = -q[i];
}

// log|det| of the factored matrix from R's diagonal (= the LU slogdet of the reference,
// np.linalg.slogdet, up to rounding): true on det == 0 or log|det| < floor.
template <class Rt>
__device__ bool volume_deficient_qr(int d, double log_floor, const Smem<Rt>& sm) {
  if (threadIdx.x < 32) {
    double l = 0.0;
    for (int j = threadIdx.x; j < d; j += 32) l += log(fabs(sm.vec[d + j]));
    l = warp_sum_d(l);
    if (threadIdx.x == 0) sm.red[2 * kWarps - 1] = l;
  }
  __syncthreads();
  return sm.red[2 * kWarps - 1] < log_floor;
}

// sum_j nu_j of the column log-norms unit_columns_regs left in sm.vec[0, d)
template <class Rt>
__device__ double col_lognorm_sum(int d, const Smem<Rt>& sm) {
  if (threadIdx.x < 32) {
    double l = 0.0;
    for (int j = threadIdx.x; j < d; j += 32) l += sm.vec[j];
    l = warp_sum_d(l);
    if (threadIdx.x == 0) sm.red[2 * kWarps - 2] = l;
  }
  __syncthreads();
  return sm.red[2 * kWarps - 2];
}

// rank-deficiency floor of the CGS2 reset (lyapunov.py:191-192): |R_jj| < 64 eps
template <class Rt>
__device__ bool rank_deficient(int d, const Smem<Rt>& sm) {
  const double tiny = 64.0 * 2.220446049250313e-16;
  bool bad = false;
  for (int j = threadIdx.x; j < d; j += kThreads) bad |= fabs(sm.vec[d + j]) < tiny;
  return __syncthreads_or(bad) != 0;
}

// the register column q (rows rc + 4i of column c) -> canonical GOOMs in out (d x d)
template <class Rt>
__device__ void export_goom(const double (&q)[16], Cx<Rt>* out, int d) {
  const ColLane L = col_lane();
  if (L.c < d)
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int r = L.rc + 4 * i;
      if (r < d) out[r * d + L.c] = cx<Rt>((Rt)log(fabs(q[i])), q[i] < 0.0 ? pi_of<Rt>() : Rt(0));
    }
}

// The policy on one state X (smem) in two halves. policy_predicate: the column norms (and
// for colinearity the Gram and the volume test) -> fire; policy_reset_value: on a fire,
// the reset value into out. The state between them (this thread's unit column, whether
// it is already factored) stays in registers. ldet_x: log|det X| when the caller tracks
// it (the walk), NaN to factor X for the volume test.
struct PolicyRun {
  double x[16];
  bool zero, factored;
};

template <class Rt>
__device__ bool policy_predicate(const Cx<Rt>* X, int d, const Policy& pol, const Smem<Rt>& sm,
                                 bool force_fire, double ldet_x, PolicyRun& st) {
  st.zero = st.factored = false;
  if (pol.kind == GOOM_POLICY_NEVER && !force_fire) return false;
  long long t0 = clock64();
  st.zero = unit_columns_regs(X, d, st.x, sm);
  prof_add(pol.timing, 2, t0);
  bool f = force_fire;
  if (pol.kind == GOOM_POLICY_NORM_THRESHOLD) {
    if (!f) {
      double m = -INFINITY;
      for (int j = threadIdx.x; j < d; j += kThreads) m = fmax(m, sm.vec[j]);
      f = block_max(m, sm.red) > pol.threshold;
    }
  } else if (pol.kind == GOOM_POLICY_COLINEARITY || force_fire) {
    f = f || st.zero;
    if (!f) {
      f = gram_offdiag_max(d, sm) > pol.threshold;
      prof_add(pol.timing, 3, t0);
    }
    if (!f && pol.log_floor != -INFINITY) {
      if (!isnan(ldet_x)) {
        // log|det| of the unit-column matrix = log|det X| - sum_j nu_j, with log|det X|
        // known from the walk (det is multiplicative): no factorisation on this path
        f = ldet_x - col_lognorm_sum(d, sm) < pol.log_floor;
      } else {
        qr_regs(st.x, d, sm);
        st.factored = true;
        f = volume_deficient_qr(d, pol.log_floor, sm);
      }
      prof_add(pol.timing, 4, t0);
    }
  }
  return f;
}

template <class Rt>
__device__ int policy_reset_value(Cx<Rt>* out, int d, const Policy& pol, const Smem<Rt>& sm,
                                  PolicyRun& st) {
  if (st.zero) return GOOM_ERANK;
  long long t0 = clock64();
  if (!st.factored) qr_regs(st.x, d, sm);
  const bool colin = pol.kind == GOOM_POLICY_COLINEARITY;
  if (colin && rank_deficient(d, sm)) return GOOM_ERANK;
  q_regs(st.x, d, colin, sm);
  prof_add(pol.timing, 5, t0);
  export_goom<Rt>(st.x, out, d);
  __syncthreads();
  prof_add(pol.timing, 6, t0);
  return GOOM_OK;
}

// both halves (the batch select / reset kernels)
template <class Rt>
__device__ int apply_policy(const Cx<Rt>* X, Cx<Rt>* out, int d, const Policy& pol,
                            const Smem<Rt>& sm, bool select_only, bool force_fire, bool* fire) {
  PolicyRun st;
  *fire = policy_predicate(X, d, pol, sm, force_fire, NAN, st);
  if (!*fire || select_only) return GOOM_OK;
  return policy_reset_value(out, d, pol, sm, st);
}

template <class C>
__device__ void copy_mat(const C* src, C* dst, int d) {
  for (int e = threadIdx.x; e < d * d; e += kThreads) dst[e] = src[e];
  __syncthreads();
}

// ---- the fused walk ----------------------------------------------------------
template <class Rt>
__global__ void __launch_bounds__(kThreads, 1)
    selective_walk_kernel(const Cx<Rt>* __restrict__ loc0, const Cx<Rt>* __restrict__ loc1,
                          Cx<Rt>* __restrict__ carries, int8_t* __restrict__ modes,
                          int64_t* __restrict__ sites, int64_t* __restrict__ n_sites,
                          int* __restrict__ status, int64_t T, int d, int s, Policy pol,
                          const double* __restrict__ ldet0, const double* __restrict__ ldet1,
                          const Rt* __restrict__ P0, const Rt* __restrict__ rs0,
                          const Rt* __restrict__ P1, const Rt* __restrict__ rs1) {
  extern __shared__ __align__(16) char smem_raw[];
  Smem<Rt> sm = carve<Rt>(smem_raw, d);
  const int64_t mat = (int64_t)d * d;
  const int64_t ntiles = (T + s - 1) / s;
  int64_t nsite = 0;
  bool have_carry = false, consumed = false;
  // log|det| of the carry (colinearity volume test): el = loc (x) carry, so
  // log|det el| = log|det loc| (batched pre-pass) + log|det carry|; a reset carry is
  // orthonormal (log|det| = 0), a kept carry is the previous el
  double ldc = 0.0;
  // left operands (tile_operand_kernel) stream into sm.tl with one bulk copy per tile,
  // issued as soon as the previous tile's predicate has released sm.R (= sm.tl)
  const uint32_t op_bytes = (uint32_t)(mat * sizeof(Rt));
  const bool bulk = P0 != nullptr && op_bytes % 16 == 0;
  const uint32_t bar = tc::smem_u32(sm.mbar);
  if (bulk && threadIdx.x == 0) {
    tc::mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0;
  bool pending = false;
  const bool tm = pol.timing != 0;
  long long t0 = clock64();
  for (int64_t k = 0; k < ntiles; ++k) {
    const int64_t lo = k * s;
    const int64_t p = (lo + s < T ? lo + s : T) - 1;
    int8_t mode;
    if (tm && threadIdx.x == 0) g_walk_prof[8] += 1;
    prof_add(tm, 7, t0);
    if (!have_carry) {
      mode = 0;
      copy_mat(loc0 + p * mat, sm.el, d);
    } else if (consumed && p == lo) {
      mode = 2;
      copy_mat(sm.carry, sm.el, d);
    } else {
      mode = consumed ? 2 : 1;
      if (P0) {
        const Rt* P = mode == 2 ? P1 : P0;
        const Rt* rs = mode == 2 ? rs1 : rs0;
        if (pending) {
          tc::mbar_wait(bar, phase);
          phase ^= 1;
          pending = false;
        } else {
          for (int64_t e = threadIdx.x; e < mat; e += kThreads) sm.tl[e] = P[k * mat + e];
        }
        for (int i = threadIdx.x; i < d; i += kThreads) sm.scal[i] = rs[k * d + i];
        prof_add(tm, 13, t0);
        lmme_right(sm.carry, sm.el, d, sm, tm);
      } else {
        block_lmme((mode == 2 ? loc1 : loc0) + p * mat, sm.carry, sm.el, d, sm);
      }
    }
    prof_add(tm, 0, t0);
    if (mode > 0)
      for (int e = threadIdx.x; e < d * d; e += kThreads) carries[k * mat + e] = sm.carry[e];
    if (threadIdx.x == 0) modes[k] = mode;
    prof_add(tm, 1, t0);
    bool fire = false;
    double ldel = NAN;
    if (ldet0) ldel = mode == 0 ? ldet0[k] : mode == 1 ? ldet0[k] + ldc : (p == lo ? ldc : ldet1[k] + ldc);
    PolicyRun st;
    if ((p % s) == s - 1 && p <= T - 2) fire = policy_predicate(sm.el, d, pol, sm, false, ldel, st);
    ldc = fire ? 0.0 : ldel;
    const bool next_consumed = fire && pol.consume != 0;
    // prefetch the next tile's left operand (sm.R is free once the predicate is done)
    if (bulk && k + 1 < ntiles) {
      const int64_t nlo = lo + s;
      const bool needs = !(next_consumed && nlo == ((nlo + s < T ? nlo + s : T) - 1));
      if (needs) {
        if (threadIdx.x == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          tc::mbar_expect_tx(bar, op_bytes);
          tc::bulk_g2s(tc::smem_u32(sm.tl), (next_consumed ? P1 : P0) + (k + 1) * mat, op_bytes, bar);
        }
        pending = true;
      }
    }
    if (tm) t0 = clock64();
    if (fire) {
      if (tm && threadIdx.x == 0) g_walk_prof[9] += 1;
      const int rc = policy_reset_value(sm.carry, d, pol, sm, st);
      if (rc != GOOM_OK) {
        if (threadIdx.x == 0) *status = rc;
        if (pending) tc::mbar_wait(bar, phase);  // no bulk copy may outlive the CTA
        break;
      }
      if (threadIdx.x == 0) sites[nsite] = p + 1;
      ++nsite;
    } else {
      Cx<Rt>* t = sm.carry;  // the kept state becomes the carry: swap buffers
      sm.carry = sm.el;
      sm.el = t;
    }
    consumed = next_consumed;
    have_carry = true;
  }
  if (threadIdx.x == 0) *n_sites = nsite;
}

// mode-2 tiles: loc0[tile] <- loc1[tile] (before materialisation)
template <class C>
__global__ void adopt_loc1_kernel(C* loc0, const C* loc1, const int8_t* modes, int64_t T, int d,
                                  int s) {
  const int64_t k = blockIdx.x;
  if (modes[k] != 2) return;
  const int64_t mat = (int64_t)d * d;
  int64_t lo = k * s, hi = lo + s < T ? lo + s : T;
  for (int64_t e = threadIdx.x; e < (hi - lo) * mat; e += blockDim.x)
    loc0[lo * mat + e] = loc1[lo * mat + e];
}

// mode-2 tiles: V[k*s] <- carry[k] (the consuming reset's own slot, scan.py:423-427)
template <class C>
__global__ void fix_reset_slots_kernel(C* V, const C* carries, const int8_t* modes, int d, int s) {
  const int64_t k = blockIdx.x;
  if (modes[k] != 2) return;
  const int64_t mat = (int64_t)d * d;
  for (int64_t e = threadIdx.x; e < mat; e += blockDim.x) V[k * s * mat + e] = carries[k * mat + e];
}

template <class Rt>
__global__ void __launch_bounds__(kThreads, 1)
    policy_select_kernel(const Cx<Rt>* X, int d, Policy pol, uint8_t* fire) {
  extern __shared__ __align__(16) char smem_raw[];
  Smem<Rt> sm = carve<Rt>(smem_raw, d);
  const int64_t mat = (int64_t)d * d;
  copy_mat(X + blockIdx.x * mat, sm.el, d);
  bool f = false;
  apply_policy(sm.el, sm.el, d, pol, sm, /*select_only=*/true, false, &f);
  if (threadIdx.x == 0) fire[blockIdx.x] = f ? 1 : 0;
}

template <class Rt>
__global__ void __launch_bounds__(kThreads, 1)
    policy_reset_kernel(const Cx<Rt>* X, Cx<Rt>* R, int d, int kind, int* status) {
  extern __shared__ __align__(16) char smem_raw[];
  Smem<Rt> sm = carve<Rt>(smem_raw, d);
  const int64_t mat = (int64_t)d * d;
  copy_mat(X + blockIdx.x * mat, sm.el, d);
  Policy pol{kind, 1, 0, 0.0, -INFINITY, 0};
  bool f = false;
  int rc = apply_policy(sm.el, R + blockIdx.x * mat, d, pol, sm, false, /*force_fire=*/true, &f);
  if (rc != GOOM_OK && threadIdx.x == 0) *status = rc;
}

// log|det| of the tiles' local products (the walk's volume test): CTA k takes the
// matrix at position min(k s + s, T) - 1 of loc; log|det| = log|det U| + sum_j nu_j with
// U the unit-column matrix (QR diagonal); -inf for a zero column.
template <class Rt>
__global__ void __launch_bounds__(kThreads, 1)
    tile_logdet_kernel(const Cx<Rt>* __restrict__ loc, int64_t T, int d, int s,
                       double* __restrict__ out) {
  extern __shared__ __align__(16) char smem_raw[];
  Smem<Rt> sm = carve<Rt>(smem_raw, d);
  const int64_t mat = (int64_t)d * d;
  const int64_t lo = (int64_t)blockIdx.x * s;
  const int64_t p = (lo + s < T ? lo + s : T) - 1;
  copy_mat(loc + p * mat, sm.el, d);
  double x[16];
  if (unit_columns_regs(sm.el, d, x, sm)) {
    if (threadIdx.x == 0) out[blockIdx.x] = -INFINITY;
    return;
  }
  const double nus = col_lognorm_sum(d, sm);
  qr_regs(x, d, sm);
  if (threadIdx.x < 32) {
    double l = 0.0;
    for (int j = threadIdx.x; j < d; j += 32) l += log(fabs(sm.vec[d + j]));
    l = warp_sum_d(l);
    if (threadIdx.x == 0) out[blockIdx.x] = l + nus;
  }
}

// Batched Householder QR with R's diagonal made non-negative (qr_factor_batched,
// lyapunov.py:79-99): one CTA per matrix, the walk's column-parallel Householder.
// from_goom: the input is a complex128 GOOM state, first log-unit-normalised per column
// (spectrum_parallel stage (b), lyapunov.py:343-347); an all-zero column sets *status.
// Outputs Q (real, row-major) and |diag R|.
// Only the reflector table and the small vectors live in shared memory (the matrix is read
// straight into registers), so several CTAs share an SM.
inline size_t qr_lean_smem_bytes(int d) {
  return ((size_t)d * d + 2 * d + 2 * kWarps + 4 * kMaxD) * sizeof(double) + 64;
}
__device__ Smem<double> carve_lean(char* base, int d) {
  Smem<double> s{};
  s.W = reinterpret_cast<double*>(base);
  s.vec = s.W + (size_t)d * d;
  s.red = s.vec + 2 * d;
  s.part = s.red + 2 * kWarps;
  return s;
}

__global__ void __launch_bounds__(kThreads, 2)
    qr_batched_kernel(const double* __restrict__ M, const double2* __restrict__ X,
                      double* __restrict__ Q, double* __restrict__ absdiag, int d,
                      int* __restrict__ status) {
  extern __shared__ __align__(16) char smem_raw[];
  Smem<double> sm = carve_lean(smem_raw, d);
  const int64_t mat = (int64_t)d * d;
  const ColLane L = col_lane();
  double x[16];
  if (X) {
    if (unit_columns_regs<double, false>(X + blockIdx.x * mat, d, x, sm)) {
      if (threadIdx.x == 0) *status = GOOM_EINVAL;
      return;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int r = L.rc + 4 * i;
      x[i] = (L.c < d && r < d) ? M[blockIdx.x * mat + r * d + L.c] : 0.0;
    }
  }
  qr_regs(x, d, sm);
  q_regs(x, d, /*positive_diag=*/true, sm);
  if (L.c < d)
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int r = L.rc + 4 * i;
      if (r < d) Q[blockIdx.x * mat + r * d + L.c] = x[i];
    }
  if (absdiag)
    for (int j = threadIdx.x; j < d; j += kThreads) absdiag[blockIdx.x * d + j] = fabs(sm.vec[d + j]);
}

inline size_t round_up(size_t x) { return (x + 255) & ~size_t(255); }

int check_policy(const goom_reset_policy* p, int d) {
  if (!p) return fail(GOOM_EINVAL, "null policy");
  if (p->check_interval < 1) return fail(GOOM_EINVAL, "check_interval must be >= 1");
  if (p->kind < GOOM_POLICY_NEVER || p->kind > GOOM_POLICY_NORM_THRESHOLD)
    return fail(GOOM_EINVAL, "unknown policy kind");
  if (d > kMaxD)
    return fail(GOOM_EUNSUPPORTED, "the fused selective walk keeps the state in one CTA: d <= 64");
  return GOOM_OK;
}

Policy to_policy(const goom_reset_policy* p) {
  static const bool timing = std::getenv("GOOM_WALK_TIMING") != nullptr;
  return Policy{p->kind, p->check_interval, p->consume_leaf, p->threshold, p->log_volume_floor,
                timing ? 1 : 0};
}

template <class Rt>
int set_smem(const void* fn, int d) {
  size_t need = smem_bytes<Rt>(d);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need) !=
      cudaSuccess)
    return cuda_fail(cudaGetLastError(), "selective smem attribute");
  return GOOM_OK;
}

// L[k*s] = skip_first ? I : A[k*s];  L[k*s+i] = A[k*s+i] (x) L[k*s+i-1]   (scan.py:317-339)
template <class Rt>
int local_products(const Cx<Rt>* A, Cx<Rt>* L, int64_t T, int d, int64_t s, bool skip_first,
                   void* lws, size_t lws_bytes, cudaStream_t st) {
  using C = Cx<Rt>;
  const int64_t mat = (int64_t)d * d;
  const int64_t nb = (T + s - 1) / s;
  if (cudaMemcpy2DAsync(L, sizeof(C) * mat * s, A, sizeof(C) * mat * s, sizeof(C) * mat, nb,
                        cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "local products copy");
  if (skip_first) GOOM_TRY(launch_identity<Rt>(L, nb, d, s * mat, st));
  for (int64_t i = 1; i < s; ++i) {
    int64_t cnt = (T - i + s - 1) / s;
    if (cnt <= 0) break;
    LmmeProblemT<Rt> p{};
    p.A = OperandT<C>{A + i * mat, s * mat, 1};
    p.B = OperandT<C>{L + (i - 1) * mat, s * mat, 1};
    p.D = OperandT<C>{nullptr, 0, 1};
    p.C = L + i * mat;
    p.strideC = s * mat;
    p.batch = cnt;
    p.n = p.k = p.m = d;
    p.rowA = ScalesT<Rt>{nullptr, 0, 1};
    p.colB = ScalesT<Rt>{nullptr, 0, 1};
    GOOM_TRY(lmme_run<Rt>(p, lws, lws_bytes, st));
  }
  return GOOM_OK;
}

template <class Rt>
size_t workspace_bytes(int64_t T, int d, const goom_reset_policy* policy) {
  if (T < 1 || d < 1 || !policy || policy->check_interval < 1) return 0;
  int64_t s = policy->check_interval < T ? policy->check_interval : T;
  int64_t nt = (T + s - 1) / s;
  size_t mat = (size_t)d * d * sizeof(Cx<Rt>);
  size_t b = round_up(mat * T);                               // loc0
  if (policy->consume_leaf && s > 1) b += round_up(mat * T);  // loc1
  b += round_up(mat * nt) + round_up(nt) + round_up(sizeof(int) * 4);
  b += 2 * round_up(sizeof(double) * (size_t)nt);             // tile log-determinants
  const int nops = policy->consume_leaf && s > 1 ? 2 : 1;     // walk left operands + scales
  b += nops * (round_up(sizeof(Rt) * (size_t)d * d * nt) + round_up(sizeof(Rt) * (size_t)d * nt));
  b += 2 * round_up(sizeof(Rt) * (size_t)T * d) + 256;        // LMME scale scratch + flag
  return b;
}

template <class Rt>
int selective_chain(const Cx<Rt>* A, Cx<Rt>* V, int64_t T, int d, const goom_reset_policy* policy,
                    int block, int64_t* sites, int64_t* n_sites, void* ws, size_t ws_bytes,
                    cudaStream_t st) {
  using C = Cx<Rt>;
  if (T < 1) return fail(GOOM_EINVAL, "scan of an empty sequence");
  if (block < 1) return fail(GOOM_EINVAL, "block_size must be >= 1");
  if (d < 1) return fail(GOOM_ESHAPE, "d must be >= 1");
  if (!A || !V || !sites || !n_sites) return fail(GOOM_EINVAL, "null pointer");
  GOOM_TRY(check_policy(policy, d));
  size_t need = workspace_bytes<Rt>(T, d, policy);
  if (ws_bytes < need || !ws) return fail(GOOM_EWORKSPACE, "selective workspace too small");
  const int64_t s = policy->check_interval < T ? policy->check_interval : T;
  const int64_t nt = (T + s - 1) / s;
  const int64_t mat = (int64_t)d * d;
  const bool need_loc1 = policy->consume_leaf && s > 1;

  char* base = reinterpret_cast<char*>(ws);
  size_t off = 0;
  C* loc0 = reinterpret_cast<C*>(base + off);
  off += round_up(sizeof(C) * mat * T);
  C* loc1 = nullptr;
  if (need_loc1) {
    loc1 = reinterpret_cast<C*>(base + off);
    off += round_up(sizeof(C) * mat * T);
  }
  C* carries = reinterpret_cast<C*>(base + off);
  off += round_up(sizeof(C) * mat * nt);
  int8_t* modes = reinterpret_cast<int8_t*>(base + off);
  off += round_up(nt);
  int* status = reinterpret_cast<int*>(base + off);
  off += round_up(sizeof(int) * 4);
  double* ldet0 = reinterpret_cast<double*>(base + off);
  off += round_up(sizeof(double) * (size_t)nt);
  double* ldet1 = reinterpret_cast<double*>(base + off);
  off += round_up(sizeof(double) * (size_t)nt);
  Rt* P0 = reinterpret_cast<Rt*>(base + off);
  off += round_up(sizeof(Rt) * (size_t)mat * nt);
  Rt* rs0 = reinterpret_cast<Rt*>(base + off);
  off += round_up(sizeof(Rt) * (size_t)d * nt);
  Rt* P1 = nullptr;
  Rt* rs1 = nullptr;
  if (need_loc1) {
    P1 = reinterpret_cast<Rt*>(base + off);
    off += round_up(sizeof(Rt) * (size_t)mat * nt);
    rs1 = reinterpret_cast<Rt*>(base + off);
    off += round_up(sizeof(Rt) * (size_t)d * nt);
  }
  void* lws = base + off;
  size_t lws_bytes = ws_bytes - off;

  // 1. local products
  GOOM_TRY(local_products<Rt>(A, loc0, T, d, s, false, lws, lws_bytes, st));
  if (need_loc1) GOOM_TRY(local_products<Rt>(A, loc1, T, d, s, true, lws, lws_bytes, st));
  // 2. fused walk
  if (cudaMemsetAsync(status, 0, sizeof(int), st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "status reset");
  GOOM_TRY(set_smem<Rt>((const void*)selective_walk_kernel<Rt>, d));
  const Policy pol = to_policy(policy);
  // the volume test's log|det| of every tile's local product, batched off the walk
  static const bool direct_volume = std::getenv("GOOM_WALK_DIRECT_VOLUME") != nullptr;
  const bool track_det = pol.kind == GOOM_POLICY_COLINEARITY && pol.log_floor != -INFINITY &&
                         !direct_volume;
  if (track_det) {
    GOOM_TRY(set_smem<Rt>((const void*)tile_logdet_kernel<Rt>, d));
    tile_logdet_kernel<Rt><<<(unsigned)nt, kThreads, smem_bytes<Rt>(d), st>>>(loc0, T, d, (int)s,
                                                                             ldet0);
    GOOM_CHECK_LAUNCH("tile_logdet_kernel");
    if (need_loc1) {
      tile_logdet_kernel<Rt><<<(unsigned)nt, kThreads, smem_bytes<Rt>(d), st>>>(loc1, T, d,
                                                                               (int)s, ldet1);
      GOOM_CHECK_LAUNCH("tile_logdet_kernel");
    }
  }
  GOOM_TRY(set_smem<Rt>((const void*)tile_operand_kernel<Rt>, d));
  tile_operand_kernel<Rt><<<(unsigned)nt, kThreads, smem_bytes<Rt>(d), st>>>(loc0, T, d, (int)s,
                                                                             P0, rs0);
  GOOM_CHECK_LAUNCH("tile_operand_kernel");
  if (need_loc1) {
    tile_operand_kernel<Rt><<<(unsigned)nt, kThreads, smem_bytes<Rt>(d), st>>>(loc1, T, d,
                                                                               (int)s, P1, rs1);
    GOOM_CHECK_LAUNCH("tile_operand_kernel");
  }
  if (pol.timing) {
    unsigned long long zero[16] = {};
    cudaMemcpyToSymbolAsync(g_walk_prof, zero, sizeof(zero), 0, cudaMemcpyHostToDevice, st);
  }
  selective_walk_kernel<Rt><<<1, kThreads, smem_bytes<Rt>(d), st>>>(
      loc0, loc1 ? loc1 : loc0, carries, modes, sites, n_sites, status, T, d, (int)s, pol,
      track_det ? ldet0 : nullptr, need_loc1 ? ldet1 : ldet0, P0, rs0, need_loc1 ? P1 : P0,
      need_loc1 ? rs1 : rs0);
  GOOM_CHECK_LAUNCH("selective_walk_kernel");
  if (pol.timing) {  // debug aid: per-phase clocks of the walk (synchronises the stream)
    unsigned long long c[16];
    cudaMemcpyFromSymbolAsync(c, g_walk_prof, sizeof(c), 0, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const char* names[10] = {"tile lmme", "carry store", "col norms", "gram", "lu volume",
                             "reset qr", "reset export", "carry copy", "tiles", "fires"};
    std::fprintf(stderr, "[walk timing] tiles %llu fires %llu:", c[8], c[9]);
    for (int i = 0; i < 8; ++i)
      std::fprintf(stderr, " %s %.1f us/tile;", names[i], c[8] ? c[i] / 1.9e3 / c[8] : 0.0);
    std::fprintf(stderr, " [lmme: operand wait %.1f, col scales + exp %.1f, gemm %.1f, log out %.1f]",
                 c[8] ? c[13] / 1.9e3 / c[8] : 0.0, c[8] ? c[10] / 1.9e3 / c[8] : 0.0,
                 c[8] ? c[11] / 1.9e3 / c[8] : 0.0, c[8] ? c[12] / 1.9e3 / c[8] : 0.0);
    std::fprintf(stderr, " (clock64 cycles / 1.9 GHz)\n");
  }
  // 3. materialise: tile 0 = loc0; tile k>0: loc[t] (x) carry[k]
  if (need_loc1) {
    adopt_loc1_kernel<C><<<(unsigned)nt, 256, 0, st>>>(loc0, loc1, modes, T, d, (int)s);
    GOOM_CHECK_LAUNCH("adopt_loc1_kernel");
  }
  const int64_t first = s < T ? s : T;
  if (cudaMemcpyAsync(V, loc0, sizeof(C) * mat * first, cudaMemcpyDeviceToDevice, st) !=
      cudaSuccess)
    return cuda_fail(cudaGetLastError(), "materialise tile 0");
  if (T > s) {
    LmmeProblemT<Rt> p{};
    p.A = OperandT<C>{loc0 + s * mat, mat, 1};
    p.B = OperandT<C>{carries + mat, mat, s};
    p.D = OperandT<C>{nullptr, 0, 1};
    p.C = V + s * mat;
    p.strideC = mat;
    p.batch = T - s;
    p.n = p.k = p.m = d;
    p.rowA = ScalesT<Rt>{nullptr, 0, 1};
    p.colB = ScalesT<Rt>{nullptr, 0, 1};
    GOOM_TRY(lmme_run<Rt>(p, lws, lws_bytes, st));
  }
  if (policy->consume_leaf) {
    fix_reset_slots_kernel<C><<<(unsigned)nt, 256, 0, st>>>(V, carries, modes, d, (int)s);
    GOOM_CHECK_LAUNCH("fix_reset_slots_kernel");
  }
  // surface a rank-deficient reset as ValueError (lyapunov.py:191-192, 212-213)
  int host_status = 0;
  if (cudaMemcpyAsync(&host_status, status, sizeof(int), cudaMemcpyDeviceToHost, st) !=
          cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "selective status read");
  if (host_status != GOOM_OK)
    return fail(host_status, "rank-deficient state cannot be orthonormalized (or all-zero column)");
  return GOOM_OK;
}

template <class Rt>
int select_batch(const void* X, int64_t batch, int d, const goom_reset_policy* policy,
                 uint8_t* fire, void* stream) {
  if (batch < 0 || d < 1) return fail(GOOM_EINVAL, "bad shape");
  GOOM_TRY(check_policy(policy, d));
  if (batch == 0) return GOOM_OK;
  GOOM_TRY(set_smem<Rt>((const void*)policy_select_kernel<Rt>, d));
  policy_select_kernel<Rt><<<(unsigned)batch, kThreads, smem_bytes<Rt>(d), as_stream(stream)>>>(
      reinterpret_cast<const Cx<Rt>*>(X), d, to_policy(policy), fire);
  GOOM_CHECK_LAUNCH("policy_select_kernel");
  return GOOM_OK;
}

template <class Rt>
int reset_batch(const void* X, void* R, int64_t batch, int d, const goom_reset_policy* policy,
                void* stream) {
  if (batch < 0 || d < 1) return fail(GOOM_EINVAL, "bad shape");
  GOOM_TRY(check_policy(policy, d));
  if (batch == 0) return GOOM_OK;
  if (policy->kind == GOOM_POLICY_NEVER) return fail(GOOM_EINVAL, "never-policy has no reset");
  cudaStream_t st = as_stream(stream);
  int* status = nullptr;
  if (cudaMallocAsync(&status, sizeof(int), st) != cudaSuccess ||
      cudaMemsetAsync(status, 0, sizeof(int), st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "reset status");
  GOOM_TRY(set_smem<Rt>((const void*)policy_reset_kernel<Rt>, d));
  policy_reset_kernel<Rt><<<(unsigned)batch, kThreads, smem_bytes<Rt>(d), st>>>(
      reinterpret_cast<const Cx<Rt>*>(X), reinterpret_cast<Cx<Rt>*>(R), d, policy->kind, status);
  GOOM_CHECK_LAUNCH("policy_reset_kernel");
  int host_status = 0;
  cudaMemcpyAsync(&host_status, status, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(status, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_fail(cudaGetLastError(), "reset sync");
  if (host_status != GOOM_OK)
    return fail(host_status, "rank-deficient state cannot be orthonormalized (or all-zero column)");
  return GOOM_OK;
}

}  // namespace
}  // namespace goom

using namespace goom;

extern "C" {

size_t goom_scan_selective_chain_workspace_size(int64_t T, int d, const goom_reset_policy* policy,
                                                int block) {
  (void)block;
  return workspace_bytes<float>(T, d, policy);
}
size_t goom_scan_selective_chain_workspace_size_c128(int64_t T, int d,
                                                     const goom_reset_policy* policy, int block) {
  (void)block;
  return workspace_bytes<double>(T, d, policy);
}
int goom_scan_selective_chain_c64(const goom_c64* A, goom_c64* V, int64_t T, int d,
                                  const goom_reset_policy* policy, int block, int64_t* sites,
                                  int64_t* n_sites, void* ws, size_t ws_bytes, void* stream) {
  return selective_chain<float>(reinterpret_cast<const float2*>(A), reinterpret_cast<float2*>(V),
                                T, d, policy, block, sites, n_sites, ws, ws_bytes,
                                as_stream(stream));
}
int goom_scan_selective_chain_c128(const goom_c128* A, goom_c128* V, int64_t T, int d,
                                   const goom_reset_policy* policy, int block, int64_t* sites,
                                   int64_t* n_sites, void* ws, size_t ws_bytes, void* stream) {
  return selective_chain<double>(reinterpret_cast<const double2*>(A),
                                 reinterpret_cast<double2*>(V), T, d, policy, block, sites,
                                 n_sites, ws, ws_bytes, as_stream(stream));
}
int goom_policy_select_c64(const goom_c64* X, int64_t batch, int d, const goom_reset_policy* policy,
                           uint8_t* fire, void* stream) {
  return select_batch<float>(X, batch, d, policy, fire, stream);
}
int goom_policy_select_c128(const goom_c128* X, int64_t batch, int d,
                            const goom_reset_policy* policy, uint8_t* fire, void* stream) {
  return select_batch<double>(X, batch, d, policy, fire, stream);
}
int goom_policy_reset_c64(const goom_c64* X, goom_c64* R, int64_t batch, int d,
                          const goom_reset_policy* policy, void* stream) {
  return reset_batch<float>(X, R, batch, d, policy, stream);
}
int goom_policy_reset_c128(const goom_c128* X, goom_c128* R, int64_t batch, int d,
                           const goom_reset_policy* policy, void* stream) {
  return reset_batch<double>(X, R, batch, d, policy, stream);
}

}  // extern "C"

namespace {
int qr_batched_entry(const double* M, const double2* X, double* Q, double* absdiag,
                     int64_t batch, int d, void* stream) {
  if (batch < 0) return goom::fail(GOOM_EINVAL, "batch must be >= 0");
  if (d < 1 || d > goom::kMaxD)
    return goom::fail(GOOM_EUNSUPPORTED, "batched QR keeps a matrix in one CTA: 1 <= d <= 64");
  if (batch == 0) return GOOM_OK;
  if ((!M && !X) || !Q) return goom::fail(GOOM_EINVAL, "null pointer");
  cudaStream_t st = goom::as_stream(stream);
  int* status = nullptr;
  if (cudaMallocAsync(&status, sizeof(int), st) != cudaSuccess ||
      cudaMemsetAsync(status, 0, sizeof(int), st) != cudaSuccess)
    return goom::cuda_fail(cudaGetLastError(), "qr status");
  if (cudaFuncSetAttribute((const void*)goom::qr_batched_kernel,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)goom::qr_lean_smem_bytes(d)) != cudaSuccess)
    return goom::cuda_fail(cudaGetLastError(), "qr smem attribute");
  goom::qr_batched_kernel<<<(unsigned)batch, goom::kThreads, goom::qr_lean_smem_bytes(d), st>>>(
      M, X, Q, absdiag, d, status);
  GOOM_CHECK_LAUNCH("qr_batched_kernel");
  int host_status = 0;
  cudaMemcpyAsync(&host_status, status, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(status, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return goom::cuda_fail(cudaGetLastError(), "qr sync");
  if (host_status != GOOM_OK)
    return goom::fail(host_status, "a scan state lost a whole column; cannot orthonormalize");
  return GOOM_OK;
}
}  // namespace

extern "C" {

int goom_qr_batched_f64(const double* M, double* Q, double* absdiag, int64_t batch, int d,
                        void* stream) {
  return qr_batched_entry(M, nullptr, Q, absdiag, batch, d, stream);
}

int goom_unit_qr_batched_c128(const goom_c128* X, double* Q, int64_t batch, int d, void* stream) {
  return qr_batched_entry(nullptr, reinterpret_cast<const double2*>(X), Q, nullptr, batch, d,
                          stream);
}

}  // extern "C"
