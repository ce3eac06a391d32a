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

#include "goom_internal.cuh"

namespace goom {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxD = 64;

struct Policy {
  int kind;
  int interval;
  int consume;
  double threshold;
  double log_floor;
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
  int* ints;      // 8
  int* iw;        // 8 + 2 * kMaxD: LU pivot partials and row permutations
};

template <class Rt>
inline size_t smem_bytes(int d) {
  size_t dd = (size_t)d * d;
  return 2 * dd * sizeof(Cx<Rt>) + 2 * dd * sizeof(double) + 2 * d * sizeof(Rt) +
         2 * d * sizeof(double) + 2 * kWarps * sizeof(double) + 4 * kMaxD * sizeof(double) +
         (16 + 2 * kMaxD) * sizeof(int) + 64;
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
  s.scal = reinterpret_cast<Rt*>(s.part + 4 * kMaxD);
  s.ints = reinterpret_cast<int*>(s.scal + 2 * d);
  s.iw = s.ints + 8;
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

// out (smem) = Lg (global, d x d) (x) Rs (smem, d x d); Eq. 10-12 at the chain's precision,
// same per-output FMA order as the SIMT kernels (bitwise-identical products).
template <class Rt>
__device__ void block_lmme(const Cx<Rt>* __restrict__ Lg, const Cx<Rt>* Rs, Cx<Rt>* out, int d,
                           const Smem<Rt>& sm) {
  const int tid = threadIdx.x, cc = tid & (kMaxD - 1), ch = tid / kMaxD;
  // clamped row maxima of Lg and column maxima of Rs: 4 row/column chunks per index
  Rt mr = Rt(-INFINITY), mc = Rt(-INFINITY);
  if (cc < d)
    for (int t = ch; t < d; t += 4) {
      mr = gmax(mr, Lg[cc * d + t].x);
      mc = gmax(mc, Rs[t * d + cc].x);
    }
  sm.part[ch * kMaxD + cc] = (double)mr;
  __syncthreads();
  if (cc < d && ch == 0)
    sm.scal[cc] = gmax(gmax(gmax((Rt)sm.part[cc], (Rt)sm.part[kMaxD + cc]),
                            gmax((Rt)sm.part[2 * kMaxD + cc], (Rt)sm.part[3 * kMaxD + cc])),
                       Rt(0));
  __syncthreads();
  sm.part[ch * kMaxD + cc] = (double)mc;
  __syncthreads();
  if (cc < d && ch == 0)
    sm.scal[d + cc] = gmax(gmax(gmax((Rt)sm.part[cc], (Rt)sm.part[kMaxD + cc]),
                                gmax((Rt)sm.part[2 * kMaxD + cc], (Rt)sm.part[3 * kMaxD + cc])),
                           Rt(0));
  __syncthreads();
  for (int e = tid; e < d * d; e += kThreads) {
    int i = e / d, j = e % d;
    Cx<Rt> z = Lg[e];  // left operand, row i, column j (= k index)
    sm.tl[j * d + i] = goom_sign_t<Rt>(z.y) * gexp(z.x - sm.scal[i]);
    Cx<Rt> q = Rs[e];  // right operand, row i (= k index), column j
    sm.tr[e] = goom_sign_t<Rt>(q.y) * gexp(q.x - sm.scal[d + j]);
  }
  __syncthreads();
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
}

// Column log-norms nu_j (FP64) into sm.vec[0..d); returns true if a column is all zero.
// Thread (column cc = tid % 64, row chunk ch = tid / 64) covers rows ch, ch+4, ...: the
// per-column max and sum of squares are 4-way partials combined through sm.part.
template <class Rt>
__device__ bool unit_columns(const Cx<Rt>* X, int d, const Smem<Rt>& sm) {
  static_assert(kThreads == 4 * kMaxD, "column-parallel mapping: 4 row chunks x 64 columns");
  const int tid = threadIdx.x, cc = tid & (kMaxD - 1), ch = tid / kMaxD;
  if (tid == 0) sm.ints[0] = 0;
  double m = -INFINITY;
  if (cc < d)
    for (int r = ch; r < d; r += 4) m = fmax(m, (double)X[r * d + cc].x);
  sm.part[ch * kMaxD + cc] = m;
  __syncthreads();
  double cm = -INFINITY;
  if (cc < d) {
    cm = fmax(fmax(sm.part[cc], sm.part[kMaxD + cc]),
              fmax(sm.part[2 * kMaxD + cc], sm.part[3 * kMaxD + cc]));
    if (cm == -INFINITY && ch == 0) sm.ints[0] = 1;
  }
  double acc = 0.0;
  if (cc < d && cm != -INFINITY)
    for (int r = ch; r < d; r += 4) acc += exp(2.0 * ((double)X[r * d + cc].x - cm));
  __syncthreads();  // every thread has read its column max before the partials are reused
  sm.part[ch * kMaxD + cc] = acc;
  __syncthreads();
  if (cc < d && ch == 0)
    sm.vec[cc] = cm == -INFINITY
                     ? -INFINITY
                     : cm + 0.5 * log(((sm.part[cc] + sm.part[kMaxD + cc]) +
                                       sm.part[2 * kMaxD + cc]) + sm.part[3 * kMaxD + cc]);
  __syncthreads();
  bool zero = sm.ints[0] != 0;
  if (!zero) {
    for (int e = tid; e < d * d; e += kThreads) {
      Cx<Rt> z = X[e];
      sm.R[e] = (double)goom_sign_t<Rt>(z.y) * exp((double)z.x - sm.vec[e % d]);
    }
  }
  __syncthreads();
  return zero;
}

// slogdet(R) via LU with partial pivoting on W; returns (det == 0) || logdet < floor.
// One barrier per pivot: rows are never swapped (a double-buffered logical -> physical
// row map instead), and the threads updating column c+1 also reduce its pivot candidates
// (4 row-chunk partials, smallest row among equal maxima, as idamax), so the next step
// starts with its pivot known. Column-parallel mapping: column cc = tid % 64 > c, logical
// rows c+1+ch, +4, ...
template <class Rt>
__device__ bool volume_deficient(int d, double log_floor, const Smem<Rt>& sm) {
  const int tid = threadIdx.x;
  const int cc = tid & (kMaxD - 1), ch = tid / kMaxD;
  double* pmax = sm.part;     // [2][4]
  int* pidx = sm.iw;          // [2][4]
  int* perm = sm.iw + 8;      // [2][kMaxD]
  for (int e = tid; e < d * d; e += kThreads) sm.W[e] = sm.R[e];
  if (tid < d) perm[tid] = tid;
  if (cc == 0) {
    double best = -1.0;
    int bi = d;
    for (int r = ch; r < d; r += 4) {
      const double v = fabs(sm.R[r * d]);
      if (v > best) { best = v; bi = r; }
    }
    pmax[ch] = best;
    pidx[ch] = bi;
  }
  __syncthreads();
  // log|det| = log(prod |pv|) kept as mantissa * 2^exponent: one log at the end, not per pivot
  double mant = 1.0;
  int expo = 0;
  for (int c = 0; c < d; ++c) {
    const int cur = c & 1, nxt = cur ^ 1;
    double best = pmax[cur * 4];
    int piv = pidx[cur * 4];
#pragma unroll
    for (int k = 1; k < 4; ++k) {
      const double v = pmax[cur * 4 + k];
      const int i = pidx[cur * 4 + k];
      if (v > best || (v == best && i < piv)) { best = v; piv = i; }
    }
    const int* pc = perm + cur * kMaxD;
    int* pn = perm + nxt * kMaxD;
    const int rowc = pc[piv];  // physical pivot row: logical row c from now on
    const int rowp = pc[c];    // physical row that moves to logical row piv
    const double pv = sm.W[rowc * d + c];
    if (pv == 0.0) return true;  // det_sign == 0 (uniform across the CTA)
    int e;
    mant = frexp(mant * fabs(pv), &e);
    expo += e;
    const double inv = 1.0 / pv;
    if (tid < d) pn[tid] = tid == c ? rowc : (tid == piv ? rowp : pc[tid]);
    double nb = -1.0;
    int ni = d;
    if (cc > c && cc < d) {
      const double u = sm.W[rowc * d + cc];
      for (int r = c + 1 + ch; r < d; r += 4) {
        const int pr = r == piv ? rowp : pc[r];
        const double nv = sm.W[pr * d + cc] - (sm.W[pr * d + c] * inv) * u;
        sm.W[pr * d + cc] = nv;
        if (cc == c + 1) {
          const double a = fabs(nv);
          if (a > nb) { nb = a; ni = r; }
        }
      }
    }
    if (cc == c + 1) {
      pmax[nxt * 4 + ch] = nb;
      pidx[nxt * 4 + ch] = ni;
    }
    __syncthreads();
  }
  return log(mant) + expo * 0.69314718055994530942 < log_floor;
}

template <class Rt>
__device__ bool policy_select(const Cx<Rt>* X, int d, const Policy& pol, const Smem<Rt>& sm) {
  if (pol.kind == GOOM_POLICY_NEVER) return false;
  bool zero = unit_columns(X, d, sm);
  if (pol.kind == GOOM_POLICY_NORM_THRESHOLD) {
    double m = -INFINITY;
    for (int j = threadIdx.x; j < d; j += kThreads) m = fmax(m, sm.vec[j]);
    return block_max(m, sm.red) > pol.threshold;
  }
  if (zero) return true;
  double g = 0.0;
  for (int e = threadIdx.x; e < d * d; e += kThreads) {
    int i = e / d, j = e % d;
    if (i >= j) continue;
    double acc = 0.0;
    for (int r = 0; r < d; ++r) acc = fma(sm.R[r * d + i], sm.R[r * d + j], acc);
    g = fmax(g, fabs(acc));
  }
  if (block_max(g, sm.red) > pol.threshold) return true;
  if (pol.log_floor == -INFINITY) return false;
  return volume_deficient(d, pol.log_floor, sm);
}

// Householder QR of sm.R in place; Q into sm.W. positive_diag flips Q columns so
// that diag(R) > 0 (the CGS2 basis). Returns GOOM_ERANK on a rank-deficient state.
template <class Rt>
__device__ int householder_q(int d, bool positive_diag, const Smem<Rt>& sm,
                             bool check_rank = true) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int cc = tid & (kMaxD - 1), ch = tid / kMaxD;  // column, row chunk (4 x 64 threads)
  double* tau = sm.vec;      // [0, d)
  double* diag = sm.vec + d;  // [d, 2d)
  for (int j = 0; j < d; ++j) {
    if (w == 0) {
      double s = 0.0;
      for (int r = j + 1 + lane; r < d; r += 32) s = fma(sm.R[r * d + j], sm.R[r * d + j], s);
      s = warp_sum_d(s);
      if (lane == 0) {
        double alpha = sm.R[j * d + j];
        if (s == 0.0) {
          tau[j] = 0.0;
          diag[j] = alpha;
          sm.red[0] = 0.0;
        } else {
          double beta = -copysign(sqrt(fma(alpha, alpha, s)), alpha);
          tau[j] = (beta - alpha) / beta;
          diag[j] = beta;
          sm.red[0] = 1.0 / (alpha - beta);
          sm.R[j * d + j] = beta;
        }
      }
    }
    __syncthreads();
    const double scale = sm.red[0];
    const double tj = tau[j];
    if (tj != 0.0) {
      if (tid > j && tid < d) sm.R[tid * d + j] *= scale;  // v_r (v_j = 1 implicit)
      __syncthreads();
      // w_c = tau (R_jc + sum_{r>j} v_r R_rc) for c > j: thread (cc, ch) sums rows j+1+ch, +4..
      double p = 0.0;
      if (cc > j && cc < d) {
        if (ch == 0) p = sm.R[j * d + cc];
        for (int r = j + 1 + ch; r < d; r += 4) p = fma(sm.R[r * d + j], sm.R[r * d + cc], p);
      }
      sm.part[ch * kMaxD + cc] = p;
      __syncthreads();
      if (cc > j && cc < d) {
        const double wc = (((sm.part[cc] + sm.part[kMaxD + cc]) + sm.part[2 * kMaxD + cc]) +
                           sm.part[3 * kMaxD + cc]) * tj;
        if (ch == 0) sm.R[j * d + cc] -= wc;
        for (int r = j + 1 + ch; r < d; r += 4) sm.R[r * d + cc] -= wc * sm.R[r * d + j];
      }
    }
    __syncthreads();
  }
  // Q = H_0 ... H_{d-1} I, accumulated backwards (LAPACK dorg2r order), same mapping
  for (int e = tid; e < d * d; e += kThreads) sm.W[e] = (e / d == e % d) ? 1.0 : 0.0;
  __syncthreads();
  for (int j = d - 1; j >= 0; --j) {
    const double tj = tau[j];
    if (tj == 0.0) continue;
    double p = 0.0;
    if (cc < d) {
      if (ch == 0) p = sm.W[j * d + cc];
      for (int r = j + 1 + ch; r < d; r += 4) p = fma(sm.R[r * d + j], sm.W[r * d + cc], p);
    }
    sm.part[ch * kMaxD + cc] = p;
    __syncthreads();
    if (cc < d) {
      const double wc = (((sm.part[cc] + sm.part[kMaxD + cc]) + sm.part[2 * kMaxD + cc]) +
                         sm.part[3 * kMaxD + cc]) * tj;
      if (ch == 0) sm.W[j * d + cc] -= wc;
      for (int r = j + 1 + ch; r < d; r += 4) sm.W[r * d + cc] -= wc * sm.R[r * d + j];
    }
    __syncthreads();
  }
  int rc = GOOM_OK;
  if (positive_diag) {
    const double tiny = 64.0 * 2.220446049250313e-16;
    if (check_rank)
      for (int j = 0; j < d; ++j)
        if (fabs(diag[j]) < tiny) rc = GOOM_ERANK;
    if (rc == GOOM_OK)
      for (int e = tid; e < d * d; e += kThreads)
        if (diag[e % d] < 0.0) sm.W[e] = -sm.W[e];
  }
  __syncthreads();
  return rc;
}

// reset(X) -> out (smem or global), canonical GOOMs. Returns a goom_status.
template <class Rt>
__device__ int policy_reset(const Cx<Rt>* X, Cx<Rt>* out, int d, int kind, const Smem<Rt>& sm) {
  bool zero = unit_columns(X, d, sm);
  if (zero) return GOOM_ERANK;
  int rc = householder_q(d, kind == GOOM_POLICY_COLINEARITY, sm);
  if (rc != GOOM_OK) return rc;
  for (int e = threadIdx.x; e < d * d; e += kThreads) {
    double q = sm.W[e];
    out[e] = cx<Rt>((Rt)log(fabs(q)), q < 0.0 ? pi_of<Rt>() : Rt(0));
  }
  __syncthreads();
  return GOOM_OK;
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
                          int* __restrict__ status, int64_t T, int d, int s, Policy pol) {
  extern __shared__ __align__(16) char smem_raw[];
  Smem<Rt> sm = carve<Rt>(smem_raw, d);
  const int64_t mat = (int64_t)d * d;
  const int64_t ntiles = (T + s - 1) / s;
  int64_t nsite = 0;
  bool have_carry = false, consumed = false;
  for (int64_t k = 0; k < ntiles; ++k) {
    const int64_t lo = k * s;
    const int64_t p = (lo + s < T ? lo + s : T) - 1;
    int8_t mode;
    if (!have_carry) {
      mode = 0;
      copy_mat(loc0 + p * mat, sm.el, d);
    } else if (consumed) {
      mode = 2;
      if (p == lo) copy_mat(sm.carry, sm.el, d);
      else block_lmme(loc1 + p * mat, sm.carry, sm.el, d, sm);
    } else {
      mode = 1;
      block_lmme(loc0 + p * mat, sm.carry, sm.el, d, sm);
    }
    if (mode > 0)
      for (int e = threadIdx.x; e < d * d; e += kThreads) carries[k * mat + e] = sm.carry[e];
    if (threadIdx.x == 0) modes[k] = mode;
    consumed = false;
    bool fire = false;
    if ((p % s) == s - 1 && p <= T - 2) fire = policy_select(sm.el, d, pol, sm);
    if (fire) {
      int rc = policy_reset(sm.el, sm.carry, d, pol.kind, sm);
      if (rc != GOOM_OK) {
        if (threadIdx.x == 0) *status = rc;
        break;
      }
      if (threadIdx.x == 0) sites[nsite] = p + 1;
      ++nsite;
      consumed = pol.consume != 0;
    } else {
      copy_mat(sm.el, sm.carry, d);
    }
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
  bool f = policy_select(sm.el, d, pol, sm);
  if (threadIdx.x == 0) fire[blockIdx.x] = f ? 1 : 0;
}

template <class Rt>
__global__ void __launch_bounds__(kThreads, 1)
    policy_reset_kernel(const Cx<Rt>* X, Cx<Rt>* R, int d, int kind, int* status) {
  extern __shared__ __align__(16) char smem_raw[];
  Smem<Rt> sm = carve<Rt>(smem_raw, d);
  const int64_t mat = (int64_t)d * d;
  copy_mat(X + blockIdx.x * mat, sm.el, d);
  int rc = policy_reset(sm.el, R + blockIdx.x * mat, d, kind, sm);
  if (rc != GOOM_OK && threadIdx.x == 0) *status = rc;
}

// Batched Householder QR with R's diagonal made non-negative (qr_factor_batched,
// lyapunov.py:79-99): one CTA per matrix, the walk's column-parallel Householder.
// from_goom: the input is a complex128 GOOM state, first log-unit-normalised per column
// (spectrum_parallel stage (b), lyapunov.py:343-347); an all-zero column sets *status.
// Outputs Q (real, row-major) and |diag R|.
__global__ void __launch_bounds__(kThreads, 1)
    qr_batched_kernel(const double* __restrict__ M, const double2* __restrict__ X,
                      double* __restrict__ Q, double* __restrict__ absdiag, int d,
                      int* __restrict__ status) {
  extern __shared__ __align__(16) char smem_raw[];
  Smem<double> sm = carve<double>(smem_raw, d);
  const int64_t mat = (int64_t)d * d;
  if (X) {
    copy_mat(X + blockIdx.x * mat, sm.el, d);
    if (unit_columns(sm.el, d, sm)) {
      if (threadIdx.x == 0) *status = GOOM_EINVAL;
      return;
    }
  } else {
    for (int e = threadIdx.x; e < d * d; e += kThreads) sm.R[e] = M[blockIdx.x * mat + e];
    __syncthreads();
  }
  householder_q(d, /*positive_diag=*/true, sm, /*check_rank=*/false);
  for (int e = threadIdx.x; e < d * d; e += kThreads) Q[blockIdx.x * mat + e] = sm.W[e];
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
  return Policy{p->kind, p->check_interval, p->consume_leaf, p->threshold, p->log_volume_floor};
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
  void* lws = base + off;
  size_t lws_bytes = ws_bytes - off;

  // 1. local products
  GOOM_TRY(local_products<Rt>(A, loc0, T, d, s, false, lws, lws_bytes, st));
  if (need_loc1) GOOM_TRY(local_products<Rt>(A, loc1, T, d, s, true, lws, lws_bytes, st));
  // 2. fused walk
  if (cudaMemsetAsync(status, 0, sizeof(int), st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "status reset");
  GOOM_TRY(set_smem<Rt>((const void*)selective_walk_kernel<Rt>, d));
  selective_walk_kernel<Rt><<<1, kThreads, smem_bytes<Rt>(d), st>>>(
      loc0, loc1 ? loc1 : loc0, carries, modes, sites, n_sites, status, T, d, (int)s,
      to_policy(policy));
  GOOM_CHECK_LAUNCH("selective_walk_kernel");
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
  GOOM_TRY(goom::set_smem<double>((const void*)goom::qr_batched_kernel, d));
  goom::qr_batched_kernel<<<(unsigned)batch, goom::kThreads, goom::smem_bytes<double>(d), st>>>(
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
