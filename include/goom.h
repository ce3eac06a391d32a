/*
 * goom.h — C ABI of the B200-native GOOM LMME prefix-scan library (libgoom.so).
 *
 * A GOOM ("generalized order of magnitude") stores a real x as the complex64
 * natural log  z = log|x| + i*pi*[x<0]; zero is (-inf, 0). Inputs may carry any
 * imaginary part: the sign is -1 iff cos(imag) < 0. Outputs are canonical
 * (imag exactly 0.0f or (float)M_PI).
 *
 * Every entry point replaces one array-level routine of the reference CPU
 * package `gooms` (/root/reference/pkg/src/gooms, cited file:line below). The
 * reference has no FFI; its boundary is the Python call surface, which the
 * Python package `paper_2510_03426_b200` re-exposes on top of this ABI (see
 * INTEGRATION.md for the ctypes binding a `gooms` maintainer would add).
 *
 * Conventions
 *   - Pointers are DEVICE pointers unless the name ends in `_host`.
 *   - Matrices are dense row-major; a batch of matrices is addressed as
 *     base + (b / div) * stride elements (stride 0 broadcasts one matrix).
 *   - All calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *     default stream) unless documented otherwise; outputs are caller-owned.
 *   - Workspace: functions taking (ws, ws_bytes) first report their need via
 *     the matching *_workspace_size() call; ws may be NULL iff that is 0.
 *   - Results are deterministic: no value-affecting atomics, fixed reduction
 *     orders; bitwise repeatable for a given argument set.
 *   - Return value: 0 = GOOM_OK, else a goom_status; goom_last_error() gives
 *     a thread-local message. Shape/argument errors map to the reference's
 *     ValueError (core.py:280-283, scan.py:40-43,94-95,518-519,539-540).
 */
#ifndef GOOM_H_
#define GOOM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct goom_c64 { float re, im; } goom_c64;
/* complex128 GOOM: float64 log-magnitude, the precision of the reference's
 * default float64 backing (core.py:189). Every _c128 entry point is the
 * FP64 twin of the _c64 one documented next to it. */
typedef struct goom_c128 { double re, im; } goom_c128;

typedef enum goom_status {
  GOOM_OK = 0,
  GOOM_EINVAL = 1,        /* bad argument (ValueError in the reference)       */
  GOOM_ESHAPE = 2,        /* dimension mismatch (ValueError)                  */
  GOOM_EDTYPE = 3,        /* unsupported element type                         */
  GOOM_ECUDA = 4,         /* CUDA runtime / launch failure                    */
  GOOM_EUNSUPPORTED = 5,  /* no sm_100a device / feature not built            */
  GOOM_EWORKSPACE = 6,    /* workspace missing or too small                   */
  GOOM_ERANK = 7          /* rank-deficient reset (lyapunov.py:191-192)       */
} goom_status;

/* ---- library ------------------------------------------------------------- */
const char* goom_last_error(void);
const char* goom_version(void);
/* 1 if `device` is an sm_100 part this build can run on, else 0. */
int goom_device_supported(int device);

/* ---- conversions (core.py:93-113, 188-239, 313-323) ------------------------ */
/* x -> (log|x|, sign); x == 0 -> (zero_log, +1).  _log_sign_arrays core.py:229-239.
 * NaN/inf inputs are NOT checked here (the Python layer raises like core.py:194-197). */
int goom_from_real_f32(const float* x, goom_c64* out, int64_t n, float zero_log, void* stream);
int goom_from_real_f64(const double* x, goom_c64* out, int64_t n, double zero_log, void* stream);
int goom_from_real_c128(const double* x, goom_c128* out, int64_t n, double zero_log, void* stream);
/* sign * exp(log), overflow -> +-inf.  GoomMatrix.to_real core.py:213-216. */
int goom_to_real_f32(const goom_c64* z, float* out, int64_t n, void* stream);
int goom_to_real_f64(const goom_c64* z, double* out, int64_t n, void* stream);
int goom_to_real_c128(const goom_c128* z, double* out, int64_t n, void* stream);
/* Per matrix b of `batch` (each `n` elements): c_b = max log (0 if all zero),
 * out = sign * exp(log - c_b + 2).  to_real_scaled core.py:313-323.
 * c is a device array of `batch` floats. */
int goom_to_real_scaled_f32(const goom_c64* z, float* out, float* c, int64_t batch, int64_t n,
                            void* stream);
int goom_to_real_scaled_c128(const goom_c128* z, double* out, double* c, int64_t batch, int64_t n,
                             void* stream);
/* SSM output export (ssm.py:84-98) straight from the chunked scan's state-assembly panels:
 * X is (H*L, d, S*nC) complex128, state (h, s, t = cc*L + i) = column s*nC + cc of matrix
 * h*L + i, t < T <= nC*L. Writes, for every state, c = max log (0 if all zero) into
 * c[(h*S + s)*T + t'] and the d-vectors log, sign and sign*exp(log - c + 2) into sl / ss / z
 * at [((h*S + s)*T + t')*d ...] (float64, (H, S, T, d)), t' = T-1-t if `reverse` else t.
 * c and z may be NULL (not written); kshift (H*S, nullable) is subtracted from the logs.
 * d <= 64, H*L <= 65535. Replaces the permute + elementwise chain after ssm_forward's scan
 * (ssm.py:84-98) and after the derived adjoint scan. */
int goom_ssm_export_c128(const goom_c128* X, int64_t H, int64_t L, int d, int64_t S, int64_t nC,
                         int64_t T, double* sl, double* ss, double* c, double* z, int reverse,
                         const double* kshift, void* stream);
/* The inverse layout: real h (H, S, T, d) float64 -> GOOM panels out (L, H, d, S*nC)
 * complex128, out[i][h][:, s*nC + cc] = from_real(h[h, s, t]) (log part + K[h,s] - c[h,s,t]
 * when K is non-NULL; c is (H, S, T)), scan time cc*L + i, t = T-1-(cc*L + i) if `reverse`.
 * T == nC*L, d <= 64. The adjoint scan's inputs without a flipped / permuted copy. */
int goom_ssm_panels_c128(const double* h, const double* K, const double* c, int64_t H, int64_t L,
                         int d, int64_t S, int64_t nC, int64_t T, int reverse, goom_c128* out,
                         void* stream);
/* The adjoint scan's source term of the SSM backward (ssm.ssm_backward_heads): per state
 * (n states of d <= 64 float64 values; sl / ss / c the forward's log, sign and per-state
 * scale, gz = C^T gy_t), z = ss * exp(sl - c + 2) and h = e^2 gz - [live] corr at i*, where
 * i* is the first index of the largest sl, corr = ss[i*] * sum_j gz_j z_j and live means some
 * sl is finite — the gradient through the shifted export's max (ssm.py:84-98). One warp per
 * state; writes h and z (n x d). */
int goom_ssm_adjoint_source_f64(const double* sl, const double* ss, const double* c,
                                const double* gz, int64_t n, int d, double* h, double* z,
                                void* stream);
/* Elementwise signed log-sum-exp, bitwise commutative.  _gadd_arrays core.py:264-275. */
int goom_gadd_c64(const goom_c64* a, const goom_c64* b, goom_c64* out, int64_t n, void* stream);
int goom_gadd_c128(const goom_c128* a, const goom_c128* b, goom_c128* out, int64_t n,
                   void* stream);
/* Per-column log Euclidean norms of batch x (rows x cols) -> batch x cols floats.
 * _col_log_norms core.py:288-296. */
int goom_col_log_norms_c64(const goom_c64* z, float* out, int64_t batch, int rows, int cols,
                           void* stream);
int goom_col_log_norms_c128(const goom_c128* z, double* out, int64_t batch, int rows, int cols,
                            void* stream);

/* ---- LMME (core.py:242-285, Eq. 10-12) ------------------------------------- */
/* C[b] = A[b] (x) B[b]  for b < batch;  A: n x k, B: k x m, C: n x m.
 * a = max(rowmax Re A, 0), b = max(colmax Re B, 0); I = (sA e^{A-a}) @ (sB e^{B-b})
 * (fp32-accurate: SIMT FP32 for small/odd shapes, 3xTF32 tcgen05 for tiles);
 * C = (log|I| + a) + b, sign(I).  Operand b addresses base + (b/div)*stride.
 * C must not alias A or B. */
typedef struct goom_operand {
  const void* ptr;  /* goom_c64* for _c64 calls, goom_c128* for _c128 calls */
  int64_t stride;  /* elements between consecutive matrices (0 = broadcast) */
  int64_t div;     /* matrix index = b / div (>= 1)                          */
} goom_operand;

size_t goom_lmme_workspace_size(int64_t batch, int n, int k, int m);
size_t goom_lmme_workspace_size_c128(int64_t batch, int n, int k, int m);
int goom_lmme_c64(goom_operand A, goom_operand B, goom_c64* C, int64_t strideC, int64_t batch,
                  int n, int k, int m, void* ws, size_t ws_bytes, void* stream);
/* Fused combine step: C[b] = (A[b] (x) B[b]) (+) D[b]   (_combine_arrays bias slot,
 * scan.py:176-177).  D.ptr == NULL behaves like goom_lmme_c64. */
int goom_lmme_gadd_c64(goom_operand A, goom_operand B, goom_operand D, goom_c64* C,
                       int64_t strideC, int64_t batch, int n, int k, int m, void* ws,
                       size_t ws_bytes, void* stream);
/* FP64 SIMT twins (complex128 GOOMs) */
int goom_lmme_c128(goom_operand A, goom_operand B, goom_c128* C, int64_t strideC, int64_t batch,
                   int n, int k, int m, void* ws, size_t ws_bytes, void* stream);
int goom_lmme_gadd_c128(goom_operand A, goom_operand B, goom_operand D, goom_c128* C,
                        int64_t strideC, int64_t batch, int n, int k, int m, void* ws,
                        size_t ws_bytes, void* stream);
/* LMME with caller-provided clamped scales (no pre-pass): rowA[(b/divA)*rowA_stride + i]
 * = max(max_j Re A[b][i][j], 0), colB[(b/divB)*colB_stride + j] likewise for the columns
 * of B (e.g. emitted by the kernel that produced the operand). No workspace. */
int goom_lmme_scaled_c64(goom_operand A, const float* rowA, int64_t rowA_stride, goom_operand B,
                         const float* colB, int64_t colB_stride, goom_c64* C, int64_t strideC,
                         int64_t batch, int n, int k, int m, void* stream);
/* Force a kernel family for testing: 0 auto, 1 SIMT, 2 tcgen05 3xTF32. Returns the
 * previous value. Process-wide. */
int goom_set_lmme_backend(int backend);
/* Engine of the complex64 chain scans for d % 256 == 0: 0 (default) the complex64 tcgen05
 * kernels with the reference's per-column clamped scales (Eq. 11) exactly; 1 the tile-scaled
 * engine (chain_ts.cu; faster, but entries more than ~e^87 below the largest of their
 * (row, 256-column block) flush). Initial value from GOOM_CHAIN_TS (=1 selects 1). Returns
 * the previous value; an out-of-range argument only queries. Process-wide. */
int goom_set_chain_engine(int engine);

/* ---- prefix scans (scan.py:181-214, 317-353, 529-563) ---------------------- */
/* Inclusive product chain out[t] = A[t] (x) ... (x) A[0] (x) carry_in, blocked exactly
 * like _scan_affine_stack's A slot (scan.py:181-214) with block = `block`:
 * products accumulate on the left. carry_in (d x d) may be NULL. */
size_t goom_scan_chain_workspace_size(int64_t T, int d, int block);
int goom_scan_chain_c64(const goom_c64* A, goom_c64* out, int64_t T, int d, int block,
                        const goom_c64* carry_in, void* ws, size_t ws_bytes, void* stream);
size_t goom_scan_chain_workspace_size_c128(int64_t T, int d, int block);
int goom_scan_chain_c128(const goom_c128* A, goom_c128* out, int64_t T, int d, int block,
                         const goom_c128* carry_in, void* ws, size_t ws_bytes, void* stream);

/* Long-chain product scan for small matrices (d <= 32, and complex64 d = 64; scan_long.cu):
 * the same prefixes out[t] = A[t] (x) ... (x) A[0] (x) carry_in as goom_scan_chain_*, for
 * chains far longer than a block, with a different but fixed combine tree (reduce-then-scan:
 * block totals, their scan by the same engine recursively, then a sequential fold of every
 * block from its carry). Sequential depth O(s log_s T) instead of the two-level tree's
 * s + T/s; 24 d^2 B of traffic per complex64 element instead of 32 d^2. Complex64
 * d = 16 / 32 / 64 fold their leaf level on tcgen05 (scan_long_tc.cu: 128 / d chains per
 * block-diagonal 3xTF32 MMA; one clamped log scale per state as the right operand);
 * otherwise every combine is the generic LMME's arithmetic, so a chain of T <= 32 is
 * bitwise the sequential fold. Replaces the block-tree A slot of _scan_affine_stack
 * (scan.py:181-214) for the long-chain harness; carry_in (d x d) may be
 * NULL. The workspace size is 0 for an unsupported d. */
size_t goom_scan_chain_long_workspace_size(int64_t T, int d);
int goom_scan_chain_long_c64(const goom_c64* A, goom_c64* out, int64_t T, int d,
                             const goom_c64* carry_in, void* ws, size_t ws_bytes, void* stream);
size_t goom_scan_chain_long_workspace_size_c128(int64_t T, int d);
int goom_scan_chain_long_c128(const goom_c128* A, goom_c128* out, int64_t T, int d,
                              const goom_c128* carry_in, void* ws, size_t ws_bytes, void* stream);

/* Inclusive affine scan of pairs (A_t: d x d, B_t: d x m, flag_t) under
 * combine_affine (scan.py:92-103): (A,B) <- (A_t A, A_t B (+) B_t), flag OR.
 * Same two-level tree as _scan_affine_stack. flags may be NULL (all false). */
size_t goom_scan_affine_workspace_size(int64_t T, int d, int m, int block);
int goom_scan_affine_c64(const goom_c64* A, const goom_c64* B, const uint8_t* flags_in,
                         goom_c64* outA, goom_c64* outB, uint8_t* flags_out, int64_t T, int d,
                         int m, int block, void* ws, size_t ws_bytes, void* stream);
size_t goom_scan_affine_workspace_size_c128(int64_t T, int d, int m, int block);
int goom_scan_affine_c128(const goom_c128* A, const goom_c128* B, const uint8_t* flags_in,
                          goom_c128* outA, goom_c128* outB, uint8_t* flags_out, int64_t T, int d,
                          int m, int block, void* ws, size_t ws_bytes, void* stream);

/* ---- selective resetting (scan.py:342-484, lyapunov.py:146-278) ------------- */
typedef enum goom_policy_kind {
  GOOM_POLICY_NEVER = 0,        /* select == false                                    */
  GOOM_POLICY_COLINEARITY = 1,  /* lyapunov.colinearity_policy: |cos| > threshold or
                                   logdet(unit-column state) < log_volume_floor;
                                   reset = CGS2 orthonormal basis (lyapunov.py:175-219) */
  GOOM_POLICY_NORM_THRESHOLD = 2 /* max column log-norm > threshold; reset = Householder
                                   Q (LAPACK sign convention) of the unit-column state
                                   (the reference scan tests' policy, test_scan.py:60-75) */
} goom_policy_kind;

typedef struct goom_reset_policy {
  int32_t kind;            /* goom_policy_kind                              */
  int32_t check_interval;  /* >= 1; tested positions p: (p+1) % interval == 0 */
  int32_t consume_leaf;    /* 1: reset value replaces the site's state        */
  int32_t reserved;
  double threshold;        /* cosine threshold or log-norm threshold          */
  double log_volume_floor; /* log(volume_floor), colinearity only             */
} goom_reset_policy;

/* Selective scan over a pure product chain: V[t] = compound state at t with
 * value-determined resets (_selective_chain_core scan.py:342-353; strided tile
 * walk for interval > 1, per-position walk for interval == 1 with tile `block`).
 * sites: device int64 array with room for T entries; n_sites: device int64.
 * Sites are identical to the sequential reference (scan.py:226-246). */
size_t goom_scan_selective_chain_workspace_size(int64_t T, int d,
                                                const goom_reset_policy* policy, int block);
int goom_scan_selective_chain_c64(const goom_c64* A, goom_c64* V, int64_t T, int d,
                                  const goom_reset_policy* policy, int block, int64_t* sites,
                                  int64_t* n_sites, void* ws, size_t ws_bytes, void* stream);
/* complex128 twin: the reference's spectrum_parallel runs this path in float64
 * (lyapunov.py:336); volume-test decisions (logdet < log 1e-9) need FP64 states. */
size_t goom_scan_selective_chain_workspace_size_c128(int64_t T, int d,
                                                     const goom_reset_policy* policy, int block);
int goom_scan_selective_chain_c128(const goom_c128* A, goom_c128* V, int64_t T, int d,
                                   const goom_reset_policy* policy, int block, int64_t* sites,
                                   int64_t* n_sites, void* ws, size_t ws_bytes, void* stream);

/* Batched policy evaluation on states X[b] (d x d): fire[b] = select(X[b]).
 * Used by the general-bias selective rounds (scan.py:255-314). */
int goom_policy_select_c64(const goom_c64* X, int64_t batch, int d, const goom_reset_policy* policy,
                           uint8_t* fire, void* stream);
/* R[b] = reset(X[b]) for the policy's reset map. */
int goom_policy_reset_c64(const goom_c64* X, goom_c64* R, int64_t batch, int d,
                          const goom_reset_policy* policy, void* stream);
int goom_policy_select_c128(const goom_c128* X, int64_t batch, int d,
                            const goom_reset_policy* policy, uint8_t* fire, void* stream);
int goom_policy_reset_c128(const goom_c128* X, goom_c128* R, int64_t batch, int d,
                           const goom_reset_policy* policy, void* stream);

/* ---- Lyapunov spectrum stages (b)-(d) (lyapunov.py:311-356) ------ */
/* Batched Householder QR of real d x d matrices (d <= 64) with R's diagonal made
 * non-negative (qr_factor_batched, lyapunov.py:79-99): Q (batch, d, d) and, if absdiag is
 * not NULL, |diag R| (batch, d). */
int goom_qr_batched_f64(const double* M, double* Q, double* absdiag, int64_t batch, int d,
                        void* stream);
/* Stage (b): each complex128 state log-unit-normalised per column, exponentiated and
 * QR-factored for its orthonormal basis Q (real). EINVAL if a state lost a whole column. */
int goom_unit_qr_batched_c128(const goom_c128* X, double* Q, int64_t batch, int d, void* stream);

/* ---- long-chain harness (SPEC.md:391-455 run_chain) -------- */
/* n random-normal reals as GOOMs, element i drawn from Philox4x32-10 keyed (seed,
 * offset + i): chain leaf t of a d x d chain uses offset t*d*d on any GPU or shard.
 * offset must be a multiple of 4. */
int goom_random_normal_c64(goom_c64* out, int64_t n, uint64_t seed, uint64_t offset,
                           void* stream);
/* Per matrix b (n elements each): out4[4b..4b+3] = {max log|x|, log ||x||_F,
 * 1 if every log-magnitude is finite or -inf else 0, 0}. */
int goom_digest_c64(const goom_c64* X, int64_t batch, int64_t n, float* out4, void* stream);
/* ---- tile-scaled fp32 chain engine (d % 256 == 0; lmme_ts.cu, chain_ts.cu) ----
 * The scan's internal matrix format: X_ij = U_ij * exp(q[i][j/256]) (U fp32 d x d,
 * q fp32 d x d/256) and G[J] = max_i q[i][J] as order-preserving uint bits (0 = unset).
 * Between scan phases no exp/log runs per element; the public complex64 chain scan
 * (goom_scan_chain_c64) imports leaves into it and exports prefixes from it. */
/* Leaves t0 .. t0+T-1 of the goom_random_normal_c64 chain, directly tile-scaled. */
int goom_random_normal_ts(float* U, float* q, uint32_t* G, int64_t T, int d, uint64_t seed,
                          uint64_t t0, void* stream);
/* complex64 (batch, rows, cols) <-> tile-scaled. */
int goom_ts_from_c64(const goom_c64* X, int64_t batch, int rows, int cols, float* U, float* q,
                     uint32_t* G, void* stream);
int goom_ts_to_c64(const float* U, const float* q, int64_t batch, int rows, int cols, goom_c64* X,
                   void* stream);
/* C[b] = A(b) (x) B(b) on tile-scaled operands (x_stride 0 broadcasts one matrix, else
 * contiguous; matrix index b / x_div). kind 0: complex64 C; 1: tile-scaled oU/oq/oG (oG
 * zero-filled by the caller); 2: digests4 (b: max log, log ||.||_F, finite, 0) with
 * parts_ws >= batch * (n/32) * (m/256) float4 of scratch. */
int goom_lmme_ts(const float* aU, const float* aq, const uint32_t* aG, int64_t a_stride,
                 int64_t a_div, const float* bU, const float* bq, const uint32_t* bG,
                 int64_t b_stride, int64_t b_div, int kind, goom_c64* C, float* oU, float* oq,
                 uint32_t* oG, float* digests4, float* parts_ws, int64_t batch, int n, int k,
                 int m, void* stream);
/* One window of the long-chain harness: the blocked chain scan (block = `block`, the
 * reference's tree, scan.py:181-214) of T tile-scaled leaves with an optional
 * tile-scaled right carry (cU/cq/cG, may be NULL); writes complex64 prefixes to `out`
 * and/or per-prefix digests (as goom_digest_c64) to digests4, and the last prefix
 * (tile-scaled) to oU/oq/oG when non-NULL. */
size_t goom_chain_ts_workspace_size(int64_t T, int d, int block);
int goom_chain_ts(const float* U, const float* q, const uint32_t* G, int64_t T, int d, int block,
                  const float* cU, const float* cq, const uint32_t* cG, goom_c64* out,
                  float* digests4, float* oU, float* oq, uint32_t* oG, void* ws, size_t ws_bytes,
                  void* stream);

/* The same window in two stages, for time-sharded runs (sharded.py): _local runs the
 * carry-independent phases 1-2 into `ws` and writes the window total (A_{T-1} ... A_0) to
 * oU/oq/oG; _finish, later and with the same ws, applies a right carry (cU/cq/cG, may be
 * NULL) to every block carry and runs phase 3 (prefixes / digests / carry-out). */
int goom_chain_ts_local(const float* U, const float* q, const uint32_t* G, int64_t T, int d,
                        int block, float* oU, float* oq, uint32_t* oG, void* ws, size_t ws_bytes,
                        void* stream);
int goom_chain_ts_finish(int64_t T, int d, int block, const float* cU, const float* cq,
                         const uint32_t* cG, goom_c64* out, float* digests4, float* oU, float* oq,
                         uint32_t* oG, void* ws, size_t ws_bytes, void* stream);

/* Snapshots of the window just scanned by goom_chain_ts / goom_chain_ts_finish with the same
 * ws: prefixes P_t (t = idx[i], window-local, host array of n), each recomputed as
 * L_t (x) carry(t / block) from the workspace (no full-window output), as complex64 into
 * out[i] and / or tile-scaled into oU/oq/oG[i] (either may be NULL, not both). */
int goom_chain_ts_snapshots(int64_t T, int d, int block, const int64_t* idx, int n,
                            goom_c64* out, float* oU, float* oq, uint32_t* oG, void* ws,
                            size_t ws_bytes, void* stream);
/* The block carries of that window (k = kidx[i], host array of n): the tile-scaled matrix
 * the engine applies on the right of block k's local products — its own P_{k block - 1}
 * (the window's carry-in for k = 0) — into oU/oq/oG[i]. */
int goom_chain_ts_carries(int64_t T, int d, int block, const int64_t* kidx, int n, float* oU,
                          float* oq, uint32_t* oG, void* ws, size_t ws_bytes, void* stream);

/* Time-sharded chain scan over an NCCL communicator (replaces the reference's
 * _scan_affine_stack A slot, scan.py:181-214, for a chain split across the GPUs of a node;
 * SURVEY §8b / §8e). Every rank passes its contiguous chunk A (T_local leaves, rank order =
 * chain order) and gets the GLOBAL prefixes of those leaves in `out`: local scan, one
 * ncclAllGather of the d x d chunk totals, the exclusive carry folded on the right, one
 * batched LMME applying it. nccl_comm is an ncclComm_t (libnccl.so.2 is resolved from the
 * process at run time); stream-ordered on `stream`. */
size_t goom_scan_chain_sharded_workspace_size(int64_t T_local, int d, int block, int nranks);
int goom_scan_chain_sharded_c64(const goom_c64* A, goom_c64* out, int64_t T_local, int d,
                                int block, void* nccl_comm, void* ws, size_t ws_bytes,
                                void* stream);
/* The same scan with digest-only output (goom_digest_c64 per global prefix into
 * digests4[4 t]): the prefixes are materialised a few blocks at a time in the workspace,
 * never all at once (config 3's 2 TiB of d = 512 prefixes). Work per rank: phases 1-2 on
 * the local chunk, one all-gather, the carry folded onto the block carries, phase 3 —
 * about two LMMEs per leaf, as on one GPU. */
size_t goom_scan_chain_sharded_digest_workspace_size(int64_t T_local, int d, int block,
                                                     int nranks);
int goom_scan_chain_sharded_digest_c64(const goom_c64* A, float* digests4, int64_t T_local, int d,
                                       int block, void* nccl_comm, void* ws, size_t ws_bytes,
                                       void* stream);

/* Profiling aid (bench.py's roofline): time every digest phase-3 launch of the
 * tile-scaled chain engine with CUDA events on its own stream. _timing(1) starts a fresh
 * log, _timing(0) stops logging; _stats synchronises and returns the logged launches,
 * their total milliseconds and total products. */
void goom_chain_ts_phase3_timing(int enable);
int goom_chain_ts_phase3_stats(int64_t* launches, double* total_ms, int64_t* products);
/* The same log per phase of a window: 0 leaf generation (goom_random_normal_ts; units =
 * leaf matrices), 1 local products (units = products), 2 block-carry fold / tree, 3 the
 * digest phase-3 launch. Each logged entry brackets all of that phase's launches. */
int goom_chain_ts_phase_stats(int phase, int64_t* launches, double* total_ms, int64_t* units);

/* Kernels libgoom has launched in this process (bench accounting). */
long long goom_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* GOOM_H_ */
