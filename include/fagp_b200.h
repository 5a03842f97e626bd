/*
 * fagp_b200.h — C ABI of the B200-native FAGP posterior (libfagp_b200.so).
 *
 * The reference (`/root/reference/pkg/src/fagp`, pure Python on numpy/OpenBLAS) has no
 * native FFI of its own: its hot path calls BLAS/LAPACK through numpy/scipy.  These entry
 * points replace exactly those call sites, one per stage of `fagp_posterior`
 * (posterior.py:267-318).  Each declaration cites the reference code it replaces.
 *
 * Conventions
 *  - Every array argument is a DEVICE pointer (row-major, float64, contiguous) unless the
 *    comment says "host".  The caller owns every buffer (inputs, outputs, workspace);
 *    the library never allocates device memory and holds no global state.
 *  - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).  All work is
 *    stream-ordered.  Only fagp_factor and fagp_read_flags synchronise `stream` (they
 *    must return a status that depends on device results).
 *  - Return value: a fagp_status.  The Python host layer maps them onto the reference's
 *    exceptions (errors.py:6-21): EINVAL -> ValueError, EBUDGET -> BudgetError,
 *    ENOTPD / ENONFINITE -> NumericalError.
 */
#ifndef FAGP_B200_H
#define FAGP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FAGP_ABI_VERSION 1
#define FAGP_MAX_P 16 /* input dimensions supported by the feature kernels */

typedef enum fagp_status {
  FAGP_OK = 0,
  FAGP_EINVAL = 1,       /* bad shape / argument            -> ValueError            */
  FAGP_EBUDGET = 2,      /* size over a configured cap      -> BudgetError           */
  FAGP_ENOTPD = 3,       /* Cholesky breakdown (+pivot)     -> NumericalError        */
  FAGP_ENONFINITE = 4,   /* non-finite feature (+row, col)  -> NumericalError        */
  FAGP_ECUDA = 5,        /* CUDA runtime / launch failure                            */
  FAGP_EWORKSPACE = 6,   /* workspace smaller than *_workspace_size()                */
  FAGP_EUNSUPPORTED = 7  /* shape outside what the kernels support (p > FAGP_MAX_P)  */
} fagp_status;

/* Device flag bits written by the feature-generating kernels (fagp_read_flags). */
#define FAGP_FLAG_X_NONFINITE 1u   /* an input coordinate is not finite  (mercer.py:334-335) */
#define FAGP_FLAG_PHI_NONFINITE 2u /* a feature value is not finite      (mercer.py:371-376) */
#define FAGP_FLAG_STALLED 4u       /* a pipelined Gram waited > ~2 s for an input chunk signal */

/*
 * Basis description: the truncated tensor-product SE eigenbasis (mercer.py:1-45).
 * `table` is a device array of fagp_basis_table_len(p, M) doubles, laid out as
 *   [0,   p)          rho_beta[d]   = rho_d * beta_d          (mercer.py:279)
 *   [p,  2p)          neg_delta2[d] = -delta2_d               (mercer.py:281, 94-99)
 *   [2p, 3p)          sqrt_beta[d]  = sqrt(beta_d)            (mercer.py:281)
 *   [3p, 3p + p*M)    lam1d[d*M+i]  = eigenvalues_1d(...)[i]  (mercer.py:146-161)
 *   [3p + p*M, +P*L)  modal[pi*L+k] = fagp_modal_coeffs(M)    (P = M(M+1)/2, L = 2M-1)
 * The shape constants are computed on the host with the reference's own scalar formulas
 * so they are bit-identical to it (shape_params, mercer.py:102-119).  m must equal M^p.
 */
typedef struct fagp_basis {
  int32_t p;           /* input dimension, 1..FAGP_MAX_P                         */
  int32_t M;           /* eigenvalues per dimension (GpModel.n_eigen)            */
  int64_t m;           /* number of tensor-product features, M^p                 */
  const double* table; /* device, see layout above                               */
} fagp_basis;

/* ---- library meta ------------------------------------------------------------------ */
int fagp_abi_version(void);
const char* fagp_strerror(int status);
int64_t fagp_basis_table_len(int32_t p, int32_t M);

/* HOST: the modal linearisation coefficients (P x L doubles, pairs a <= b a-major):
 * h_a(z) h_b(z) = sum_k V[pi][k] h_k(sqrt(2) z), h = the reference's normalised Hermite
 * polynomials (mercer.py:122-143).  Products of two eigenfunctions of one dimension then
 * lie in the span of L = 2M-1 functions g_k = beta e^{-2 delta2 x^2} h_k(sqrt2 rho beta x),
 * which is what lets the Gram and variance kernels contract over L^p instead of P^p
 * columns.  Exact identity (long-double recurrence, |V| <= 1). */
int fagp_modal_coeffs(int32_t M, double* out_host);

/* Multi-index enumeration, HOST output (m x p int64, 1-based, first dimension slowest).
 * Replaces mercer.multi_indices (mercer.py:195-216); bit-exact with it. */
int fagp_multi_indices(int32_t M, int32_t p, int64_t* out_host);

/* Copy the device flag word to the host (synchronises stream) and clear it. */
int fagp_read_flags(uint32_t* flags_dev, uint32_t* flags_host, void* stream);

/* ---- (1) eigen-decomposition ------------------------------------------------------- */
/* Product eigenvalues lam[j] = ((1*lam1[i1])*lam2[i2])*...  (mercer.py:350-353),
 * the floored copy max(lam, max(lam)*floor_rel) (mercer.py:259-266) and its square root
 * s = sqrt(lam_floored) (posterior.py:169-170).  Any output may be NULL. */
int fagp_eigenvalues(const fagp_basis* basis, double floor_rel, double* lam, double* lam_floored,
                     double* sqrt_lam, void* stream);

/* Normalized Hermite values h_k(z), k < count (mercer.py:122-143).  out: n x count. */
int fagp_hermite(const double* z, int64_t n, int32_t count, double* out, void* stream);

/* Table rows.  Row r of a table T (N x W, W = fagp_table_width(p, M)) holds
 *   [d*M + i]  (sqrt_beta_d * exp((-delta2_d * x) * x)) * h_i((rho_d beta_d) * x), x = X[r, d]
 *              -- the per-dimension eigenfunctions, _phi_1d (mercer.py:276-281)
 *   [p*M]      r = y[r] - mean_const (posterior.py:229), 0 when y is NULL
 *   [p*M + 1]  1.0      [p*M + 2]  0.0      [p*M + 3 .. W)  0.0 (pad to an even width)
 * so every column of [Phi | r | 0] is a product of p entries of one row. */
int32_t fagp_table_width(int32_t p, int32_t M);

/* Evaluate the table for every row of X (N x p).  Sets FAGP_FLAG_X_NONFINITE in *flags
 * (nullable) when an input coordinate is not finite (mercer.py:334-335). */
int fagp_basis_eval(const double* X, int64_t N, const fagp_basis* basis, const double* y,
                    double mean_const, double* T, uint32_t* flags, void* stream);

/* Rewrite the residual column of an existing table: T[r, p*M] = y[r] - mean_const. */
int fagp_set_residual(double* T, int64_t N, const fagp_basis* basis, const double* y, double mean_const,
                      void* stream);

/* ---- (2) feature matrix ------------------------------------------------------------ */
/* Materialise Phi (N x m) from the table T (mercer.py:284-292).  Not on the posterior
 * path (the Gram and predict kernels generate Phi tiles on chip); kept for the
 * EigenSystem.phi attribute and for parity tests. */
int fagp_features(const double* T, int64_t N, const fagp_basis* basis, double* phi,
                  uint32_t* flags, void* stream);

/* Locate the first non-finite Phi entry in row-major order (np.argwhere(~isfinite(phi))[0],
 * mercer.py:371-376) without materialising Phi.  *first_dev (device int64) receives
 * row * m + col, or -1 when every feature is finite. */
int fagp_find_nonfinite(const double* T, int64_t N, const fagp_basis* basis, int64_t* first_dev,
                        void* stream);

/* Fused feature generation + Gram contraction on FP64 tensor cores (DMMA).
 * Replaces `backend.gemm(phi, phi, transpose_a=True)` (posterior.py:168) and
 * `backend.gemm(phi, y - c, transpose_a=True)` (posterior.py:229,233), with Phi never
 * written to HBM.  The output `gram` (fagp_gram_len(basis) doubles) is a compressed form
 * of G = Phi^T Phi and t = Phi^T (y - c), read by fagp_factor / fagp_gram_unpack:
 *  - 2 <= p <= 8 ("modal form"): [K | t].  Every product phi_d,a phi_d,b of one dimension is
 *    an exact combination of L = 2M-1 functions g_d,k (fagp_modal_coeffs), so
 *    G[(a),(a')] = sum_kappa K[kappa] prod_d V[{a_d,a'_d}][kappa_d] with
 *    K[kappa] = sum_r prod_d g_d,kappa_d(x_rd): L^p entries (first dimension slowest), one
 *    rectangular DMMA GEMM over the rows; t = Phi^T r (m entries, canonical feature order)
 *    comes out of the same launch.
 *  - p == 1: the packed upper triangle of [Phi | r]^T [Phi | r] ((m+1)(m+2)/2, row-major;
 *    column m holds t), from a fused SYRK.
 * This buffer is also the only data multi-GPU callers all-reduce (sum over row shards).
 * Deterministic for fixed (N, basis): fixed split-K trees, no floating-point atomics.
 * T comes from fagp_basis_eval(X, y, mean_const).  Sets FAGP_FLAG_PHI_NONFINITE when a
 * feature is not finite (detected on the Gram entries). */
int64_t fagp_gram_len(const fagp_basis* basis);
size_t fagp_gram_workspace_size(int64_t N, const fagp_basis* basis);
int fagp_gram(const double* T, int64_t N, const fagp_basis* basis, double* gram, void* workspace,
              size_t workspace_bytes, uint32_t* flags, void* stream);

/* The same `gram` buffer straight from the points: X (N x p) and y (N, nullable: t = 0),
 * r = y - mean_const (posterior.py:229).  For the modal shapes whose output fits one CTA's
 * registers (p <= 4, e.g. BASELINE C2/C3) the 1-D eigenfunctions are evaluated on chip by
 * producer warps and no basis table ever reaches HBM (fused.cu); other shapes evaluate a
 * table into the workspace and run fagp_gram.  Same output, determinism and flags as
 * fagp_gram (FAGP_FLAG_X_NONFINITE for a non-finite coordinate, mercer.py:334-335). */
size_t fagp_gram_x_workspace_size(int64_t N, const fagp_basis* basis);
int fagp_gram_x(const double* X, int64_t N, const fagp_basis* basis, const double* y, double mean_const,
                double* gram, void* workspace, size_t workspace_bytes, uint32_t* flags, void* stream);

/* The same call split into fagp_gram_x_chunks(N, basis) launches so a host pipeline can
 * overlap the upload of the rows with the contraction: every CTA owns a contiguous row range
 * cut into that many sub-ranges, chunk k contracts sub-range k of every CTA (all SMs busy),
 * and fagp_gram_x_upload_chunk(k) is the matching H2D copy (HOST X_host / y_host, pinned for
 * an asynchronous copy; one 2-D cudaMemcpy per array).  Chunks are issued in order on one
 * stream; the last one writes `gram`.  Deterministic (per (CTA, sub-range) partials summed in
 * a fixed order); equal to fagp_gram_x within rounding (fagp_gram_x keeps one partial per CTA).
 * Table-path shapes: 1 chunk. */
int32_t fagp_gram_x_chunks(int64_t N, const fagp_basis* basis);
int fagp_gram_x_upload_chunk(const double* X_host, const double* y_host, int64_t N, const fagp_basis* basis,
                             int32_t k, double* X, double* y, void* stream);
int fagp_gram_x_chunk(const double* X, int64_t N, const fagp_basis* basis, const double* y, double mean_const,
                      int32_t k, double* gram, void* workspace, size_t workspace_bytes, uint32_t* flags,
                      void* stream);

/* The pipelined form: ONE fused Gram launch that overlaps the uploads.  Before contracting
 * sub-range k, its CTAs wait (acquire) for ready[k] != 0; the host issues, on a copy stream,
 * fagp_gram_x_upload_chunk(k) followed by fagp_gram_x_signal(ready, k) (a 4-byte
 * stream-ordered H2D copy -- a copy engine, not a kernel, so it runs beside the waiting Gram).
 * `ready` is fagp_gram_x_chunks(N, basis) zeroed device words; the launch re-arms them (zeroes
 * them after the Gram).  Bitwise identical to fagp_gram_x.  A signal that never comes raises
 * FAGP_FLAG_STALLED after ~2 s instead of hanging.  Fused shapes only (else FAGP_EUNSUPPORTED). */
int fagp_gram_x_pipelined(const double* X, int64_t N, const fagp_basis* basis, const double* y, double mean_const,
                          uint32_t* ready, double* gram, void* workspace, size_t workspace_bytes, uint32_t* flags,
                          void* stream);
int fagp_gram_x_signal(uint32_t* ready, int32_t k, void* stream);

/* Expand a `gram` buffer into the full symmetric G (m x m, nullable) and t (m, nullable).
 * The modal form needs fagp_gram_unpack_workspace_size(basis) bytes of workspace for G. */
size_t fagp_gram_unpack_workspace_size(const fagp_basis* basis);
int fagp_gram_unpack(const double* gram, const fagp_basis* basis, double* G, double* t, void* workspace,
                     size_t workspace_bytes, void* stream);

/* ---- (3) Cholesky factorisation and solves ----------------------------------------- */
/* Scaled system A = (s_i G_ij) s_j + sigma2 I (posterior.py:171-174) from the `gram` buffer,
 * its Cholesky factor with the reference's jitter schedule [0, b, 10b, 100b],
 * b = 1e-12 trace(A)/m (backend.py:154-189), V = L^{-1} diag(s) (TRTRI), the mean weights
 * w = V^T V t = s * A^{-1}(s * t) (posterior.py:233-235) and the predict operand
 * (pair form: [Ct | w] with Ct the pair-folded S A^{-1} S; p == 1: [V^T | w]).
 * Synchronises `stream` once per attempt.  Outputs (device): L (m x m, lower; upper part
 * zeroed), G (m x m symmetric, nullable), t (m), w (m), predict_op
 * (fagp_predict_operand_len(basis) doubles, nullable).  Host outputs: *jitter (the jitter
 * that succeeded), *pivot_index (1-based LAPACK-style leading minor on ENOTPD, else 0). */
size_t fagp_factor_workspace_size(int64_t m);
int64_t fagp_predict_operand_len(const fagp_basis* basis);
int fagp_factor(const double* gram, const fagp_basis* basis, const double* sqrt_lam, double sigma2,
                int32_t jitter_attempts, double* L, double* G, double* t, double* w, double* predict_op,
                double* jitter, int32_t* pivot_index, void* workspace, size_t workspace_bytes,
                void* stream);

/* fagp_factor for the modal shapes (2 <= p <= 8) without the Cholesky factor: the same A, jitter
 * schedule, pivot_index on breakdown, G, t, w and predict operand, with A^{-1} (m x m, full
 * symmetric, required) from ONE persistent cooperative kernel -- the right-looking blocked
 * Cholesky of fagp_potrf (same pivot test and LAPACK info), the triangular inverse eliminated
 * in the same 32-column steps, and X^T X -- instead of ~2 m/32 + 12 launches.  The posterior
 * hot path needs only A^{-1} (posterior.py:233-235, 252-262).  FAGP_EUNSUPPORTED for p == 1
 * and for m > 2048, where the blocked route wins (use fagp_factor).  Same workspace as
 * fagp_factor. */
int fagp_factor_inv(const double* gram, const fagp_basis* basis, const double* sqrt_lam, double sigma2,
                    int32_t jitter_attempts, double* Ainv, double* G, double* t, double* w, double* predict_op,
                    double* jitter, int32_t* pivot_index, void* workspace, size_t workspace_bytes, void* stream);

/* Attempt 0 of fagp_factor_inv (no jitter) enqueued with NO host synchronisation: every kernel
 * is issued unconditionally and the breakdown index is copied asynchronously to *info_host
 * (HOST, pinned; valid once `stream` has synchronised).  Lets a caller queue the prediction right
 * behind the factor so the GPU never waits for the host.  If *info_host != 0 the outputs are
 * invalid and the caller must run fagp_factor_inv (the full jitter schedule) and redo the
 * prediction; with sigma2 > 0 this does not happen for data that does not need jitter. */
int fagp_factor_inv_async(const double* gram, const fagp_basis* basis, const double* sqrt_lam, double sigma2,
                          double* Ainv, double* G, double* t, double* w, double* predict_op, int32_t* info_host,
                          void* workspace, size_t workspace_bytes, void* stream);

/* Overwrite the mean weights stored in the predict operand with w (used after the
 * reference's fault-injection hook flips w, posterior.py:245-246). */
int fagp_set_mean_weights(double* predict_op, const double* w, const fagp_basis* basis, void* stream);

/* Plain lower Cholesky of a symmetric m x m matrix, in place, no jitter: the single
 * dpotrf call inside SpdFactor (backend.py:172).  *info_dev (device int32) receives 0 or
 * the 1-based index of the first non-positive pivot.  Upper part is left untouched. */
size_t fagp_potrf_workspace_size(int64_t m);
int fagp_potrf(double* A, int64_t m, int32_t* info_dev, void* workspace, size_t workspace_bytes,
               void* stream);

/* Inverse of a symmetric positive definite m x m matrix (dpotrf + dpotri) by fagp_factor_inv's
 * persistent kernel: Ainv (full symmetric) = A^{-1}; A is overwritten.  *info_dev
 * (device int32) = 0, or the 1-based column where dpotrf would report the matrix not positive
 * definite (Ainv is then unspecified).  A and Ainv must not alias. */
size_t fagp_spd_inverse_workspace_size(int64_t m);
int fagp_spd_inverse(double* A, int64_t m, double* Ainv, int32_t* info_dev, void* workspace, size_t workspace_bytes,
                     void* stream);

/* cho_solve (backend.py:191-193): B <- A^{-1} B given the lower factor L; B is m x nrhs. */
int fagp_potrs(const double* L, int64_t m, double* B, int64_t nrhs, void* stream);

/* General FP64 DMMA GEMM, C = alpha op(A) op(B) + beta C, row-major (op = transpose when
 * trans_* != 0).  Backs Backend.gemm (backend.py:90-130) and the optional full covariance
 * (posterior.py:258-263) -- neither is on the mean/variance path. */
int fagp_dgemm(int32_t trans_a, int32_t trans_b, int64_t M, int64_t N, int64_t K, double alpha,
               const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
               int64_t ldc, void* stream);

/* V = L^{-1} diag(s) (lower triangular; s may be NULL for L^{-1}).  Replaces the
 * covariance inner matrix solve_inner(I) (posterior.py:252-255) in restated form. */
size_t fagp_trtri_workspace_size(int64_t m);
int fagp_trtri(const double* L, const double* s, int64_t m, double* V, void* workspace,
               size_t workspace_bytes, void* stream);

/* ---- (4) predictive mean and variance ---------------------------------------------- */
/*   mean[i] = mean_const + Phi*_i . w                   (posterior.py:247)
 *   var[i]  = sigma2 * phi*_i^T (S A^{-1} S) phi*_i      (= diag of posterior.py:249-263,
 *                                                          the variance cli.py:222 reports)
 * Pair form (p >= 2): var = sigma2 sum_pi Ct[pi] prod_d q_d[i, pi_d] as a DMMA GEMM over the
 * pair combos with a fused q-product epilogue; mean by nested per-dimension sums.
 * p == 1: fused Phi*-generation + DMMA contraction with [V^T | w] + row sums of squares.
 * Ts = fagp_basis_eval(Xstar).  var may be NULL (mean only). */
int fagp_predict(const double* Ts, int64_t Ns, const fagp_basis* basis, const double* predict_op,
                 double sigma2, double mean_const, double* mean, double* var, uint32_t* flags,
                 void* stream);

/* fagp_predict straight from the test points Xs (Ns x p): mean and variance
 * (posterior.py:247, 249-263 diagonal) in one fused pass -- producer warps evaluate the
 * eigenfunctions on chip, the variance operand and mean weights sit in shared memory, and
 * both contractions run on the DMMA pipe (fused.cu) -- for the modal shapes whose operand
 * fits shared memory (p <= 4, M <= 24, e.g. BASELINE C2/C3); other shapes evaluate a table
 * into the workspace (fagp_predict_x_workspace_size bytes, 0 on the fused path) and run
 * fagp_predict.  var may be NULL. */
/* Rows one full wave of the fused predict covers (SMs x rows per block; 0 for table-path
 * shapes): a host pipeline that predicts in chunks cuts them at multiples of this, so only the
 * last chunk has a partial wave. */
int64_t fagp_predict_x_wave_rows(const fagp_basis* basis);
/* Which kernels the point-input entries run for this shape (no compute, no device needed):
 * out[0] = fagp_gram_x route, out[1] = fagp_predict_x route (0: basis table + tiled table kernels,
 * 1: one-CTA fused kernel, 2: output-tiled fused kernel), out[2] = factor route (0: fagp_factor,
 * blocked potrf + trtri + lauum; 1: fagp_factor_inv, the persistent Cholesky inverse).
 * Diagnostics / bench accounting; replaces nothing in the reference. */
int fagp_route_info(int64_t N, int64_t Ns, const fagp_basis* basis, int32_t* out);
/* HOST memcpy (dst pinned staging buffer, src the caller's pageable array) over `threads` threads
 * with non-temporal stores, so the H2D DMA that follows reads DRAM rather than dirty CPU cache
 * lines.  The staging step of fagp_posterior's host path for numpy inputs (posterior.py:267-318
 * takes numpy arrays); no device work. */
int fagp_host_copy(void* dst, const void* src, size_t bytes, int32_t threads);
/* 1 when [p, p + bytes) is pinned host memory the device can access at the same address (mapped
 * under unified addressing), else 0: fagp_predict_x's mean / var may then point straight into it
 * (zero-copy results: the kernel's stores cross PCIe as it runs, no D2H copy follows).  No device
 * work. */
int fagp_host_mapped(const void* p, size_t bytes);
int fagp_host_copy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                      int32_t threads);
/* Host staging of exactly the rows fagp_gram_x_upload_chunk(k) will copy: from the caller's
 * pageable X_src / y_src (N x p, N) into pinned X_pinned / y_pinned laid out like X / y, with
 * fagp_host_copy's threads and streaming stores -- so chunk k can be staged while chunk k-1 is
 * in flight (the numpy-input host path of posterior.py:267-318). */
int fagp_gram_x_stage_chunk(const double* X_src, const double* y_src, int64_t N, const fagp_basis* basis, int32_t k,
                            double* X_pinned, double* y_pinned, int32_t threads);
size_t fagp_predict_x_workspace_size(int64_t Ns, const fagp_basis* basis);
int fagp_predict_x(const double* Xs, int64_t Ns, const fagp_basis* basis, const double* predict_op,
                   double sigma2, double mean_const, double* mean, double* var, uint32_t* flags,
                   void* workspace, size_t workspace_bytes, void* stream);

/* ---- (6) method="literal": the reference's cross-check route ---------------------------
 * posterior.py:236-244 (mean through t1..t5) and 256-260 (inner covariance).  Built from
 * the Gram/predict kernels above plus these pieces; the Python host (posterior.py in this
 * package) strings them together exactly as the reference's expressions are ordered. */

/* y = mean_const + Phi x over the rows of a table (backend.gemm(phi, x), posterior.py:241,247).
 * Phi generated on chip from T; any 1 <= p <= 8.  Sets FAGP_FLAG_PHI_NONFINITE on a
 * non-finite output. */
int fagp_phi_matvec(const double* T, int64_t N, const fagp_basis* basis, const double* x,
                    double mean_const, double* y, uint32_t* flags, void* stream);

/* out = Phi^T v (backend.gemm(phi, v, transpose_a=True), posterior.py:240,243).  Writes v
 * into T's residual column (T is modified), then runs the Gram kernel's t-tiles only. */
size_t fagp_phi_tmatvec_workspace_size(int64_t N, const fagp_basis* basis);
int fagp_phi_tmatvec(double* T, int64_t N, const fagp_basis* basis, const double* v, double* out,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Elementwise vector ops, numpy rounding (one IEEE op per numpy operator). */
#define FAGP_VEC_DIV 0        /* out = x / alpha         t1 = r / sigma2 (posterior.py:239) */
#define FAGP_VEC_SUB_DIV 1    /* out = x - y / alpha     t5 = t1 - t4 / sigma2 (:242)       */
#define FAGP_VEC_MUL 2        /* out = x * y             w = lam_f * u (:244)               */
#define FAGP_VEC_SUB 3        /* out = x - y             mid = g - g @ solve(g) (:258)      */
#define FAGP_VEC_SUB_SCALAR 4 /* out = x - alpha         r = y - mean_const (:229)          */
int fagp_vec_op(int32_t op, int64_t n, const double* x, const double* y, double alpha, double* out,
                void* stream);

/* LambdaBarSolve.matrix (posterior.py:184-188): 0.5 (B + B^T), B = diag(1/lam_f) + G/sigma2.
 * G, out: m x m (distinct buffers). */
int fagp_lambda_bar(const double* G, const double* lam_f, int64_t m, double sigma2, double* out,
                    void* stream);

/* inner = 0.5 (A + A^T), A = diag(lam_f) - lam_f[:, None] * mid * lam_f[None, :]
 * (posterior.py:259-261).  mid, inner: m x m (distinct buffers). */
int fagp_literal_inner(const double* mid, const double* lam_f, int64_t m, double* inner,
                       void* stream);

/* A fagp_predict operand (fagp_predict_operand_len doubles) for an explicit inner matrix:
 * fagp_predict(..., sigma2 = 1.0, ...) then returns var_i = phi*_i^T inner phi*_i and
 * mean_i = mean_const + phi*_i . w.  Modal form (2 <= p <= 8) only: FAGP_EUNSUPPORTED
 * otherwise (use fagp_features + fagp_dgemm + fagp_rowdot), returned before the pointer
 * checks so a call with NULL pointers probes the form. */
size_t fagp_inner_operand_workspace_size(const fagp_basis* basis);
int fagp_inner_operand(const double* inner, const double* w, const fagp_basis* basis,
                       double* predict_op, void* workspace, size_t workspace_bytes, void* stream);

/* out[i] = sum_j A[i, j] B[i, j] (A, B: n x k) -- diag(Phi* inner Phi*^T) from
 * B = Phi* inner (posterior.py:262, cli.py:222). */
int fagp_rowdot(const double* A, const double* B, int64_t n, int64_t k, double* out, void* stream);

/* ---- the exact dense GP (validation route) ------------------------
 * K[i, j] = exp(-sum_d (eps_d (A[i, d] - B[j, d]))^2) (+ diag_add on i == j): the reference's
 * gram_matrix (kernels.py:119-145) with its accumulation order, and with diag_add = sigma2 the
 * C = K + sigma2 I of exact_posterior (posterior.py:131-132).  A (na x p), B (nb x p) row-major
 * device points; eps_host: p host doubles (p <= 64); K row-major with leading dimension ldk.
 * exact_posterior then runs on fagp_potrf (jitter on the host), fagp_potrs and fagp_dgemm. */
int fagp_se_gram(const double* A, int64_t na, const double* B, int64_t nb, int32_t p, const double* eps_host,
                 double diag_add, double* K, int64_t ldk, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FAGP_B200_H */
