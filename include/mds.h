/*
 * mds.h — C-ABI of the B200-native condensed-KKT hot path of the mixed
 * dense-sparse (MDS) interior-point method (arxiv/paper_2605_13736,
 * PAPER.md §2, "Porting the Nonlinear Optimization Library HiOp to
 * Accelerator-Based Hardware Architectures").
 *
 * One Newton iteration's KKT work (Fig.1):
 *   mds_condense     Eq.(5) -> Eq.(6): eliminate the diagonal sparse block
 *                    (K3 "M := M + A D B^T") -> dense M, rhs_c
 *   mds_factor       Bunch-Kaufman LDL^T of M with inertia (K4)
 *   mds_solve        forward/backward solves + sparse-step recovery (K4 + K2)
 *   ipm_step_vectors fraction-to-boundary + norms (K1)
 *
 * ---------------------------------------------------------------------------
 * Conventions (apply to every entry point)
 *  - All pointers named *_dev or documented "device" are CUDA device pointers
 *    owned by the CALLER; the library allocates nothing inside the hot calls
 *    (only mds_plan_create allocates, for the pattern-derived index maps).
 *  - Dense symmetric matrices are column-major with leading dimension ld >= N;
 *    only the LOWER triangle is read or written (LAPACK uplo='L').  Element
 *    (i,j), i >= j, is at A[i + j*ld].
 *  - J_s is CSR n_s x m with ROWS = sparse variables (reading R1 in DESIGN.md):
 *    row k lists the constraints sparse variable k enters; column c < m_E is an
 *    equality row g of Eq.(5), c >= m_E an inequality row h.  CSR must be
 *    canonical (sorted, unique column indices per row).
 *  - Unknown order of M / rhs_c / dxy is (x_d, y_g, y_h), as Eq.(6)
 *    (PAPER.md:169-176).  N = n_d + m_E + m_I.
 *  - `stream` is a cudaStream_t passed as void*.  Every call is asynchronous
 *    and stream-ordered, except mds_factor with inertia_host != NULL, which
 *    synchronises the stream to return the inertia (the IPM must branch on it,
 *    PAPER.md:161).
 *  - Return value: MDS_OK, or an argument error detected on the host
 *    (MDS_ERR_ARG / MDS_ERR_PATTERN / MDS_ERR_WORKSPACE) or a CUDA launch error
 *    (MDS_ERR_CUDA).  Data-dependent errors are written to *status_dev (a
 *    device int32 the caller zeroes; the first error wins).
 *  - FP64 throughout.
 * ---------------------------------------------------------------------------
 */
#ifndef MDS_B200_H
#define MDS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MDS_OK = 0,
    MDS_ERR_ARG = -1,          /* null pointer, negative size, ld < N          */
    MDS_ERR_PATTERN = -2,      /* CSR unsorted / duplicate / out of range      */
    MDS_ERR_NONPOSITIVE = -3,  /* q_k = h_ss+sigma_s+delta_w <= 0 or d_h <= 0  */
    MDS_ERR_NONFINITE = -4,    /* NaN/Inf in M before factoring                */
    MDS_ERR_SINGULAR = -5,     /* zero 1x1 pivot (|d| <= tol) met by the solve */
    MDS_ERR_NOT_INTERIOR = -6, /* x not strictly inside a finite bound, z <= 0 */
    MDS_ERR_CUDA = -7,         /* CUDA launch / runtime error                  */
    MDS_ERR_WORKSPACE = -8     /* workspace too small                          */
} mds_status;

/* Inertia triple (positive, zero, negative eigenvalue counts). */
typedef struct {
    int64_t pos, zero, neg;
} mds_inertia;

/* Opaque, immutable per-sparsity-pattern plan (the pattern is fixed across IPM
 * iterations).  Holds device copies of the CSR pattern of J_s and its
 * constraint-major transpose map.  Shareable across streams. */
typedef struct mds_plan mds_plan;

/* Library version string, e.g. "mds_b200 0.1 sm_100a". */
const char *mds_version(void);

/* Build a plan from the HOST CSR pattern of J_s (rowptr[n_s+1], colidx[nnz]).
 * Validates the pattern (MDS_ERR_PATTERN) and uploads index maps to the
 * current device.  *out receives the plan. */
int mds_plan_create(int64_t n_s, int64_t n_d, int64_t m_E, int64_t m_I,
                    const int32_t *rowptr_host, const int32_t *colidx_host, mds_plan **out);
int mds_plan_destroy(mds_plan *plan);
/* Dimensions of a plan: out[0..4] = n_s, n_d, m_E, m_I, nnz. */
int mds_plan_dims(const mds_plan *plan, int64_t *out5);

/* ---------------------------------------------------------------------------
 * mds_condense — Eq.(5) -> Eq.(6) with the regularisation
 * of PAPER.md:161 folded in:
 *   q_k   = h_ss[k] + sigma_s[k] + delta_w ;  w_k = 1/q_k         (Q_{x_s}^{-1})
 *   M_xx  = H_dd + diag(sigma_d) + delta_w I                        (block (1,1))
 *   M_yx  = J_d                                                     (blocks (2,1),(3,1))
 *   M_yy  = -J_s^T diag(w) J_s - diag(0_{m_E}, 1/d_h) - delta_c I   (blocks (2,2)..(3,3))
 *   rhs_c = [ r_xd ; r_y - J_s^T (w .* r_xs) ]
 * plus, fused into the stores, the pre-factor scan of SURVEY §8(a3):
 *   anorm_out = ||M||_inf (row abs-sums of the symmetric M from its lower
 *   triangle, fixed summation order -> bitwise reproducible), or NaN if M
 *   holds a NaN/Inf entry.  Feed it to mds_factor's `anorm` to skip its scan.
 * w is formed with the elimination's own operations (IEEE division).  The
 * products (val_p w_k) val_p' of each entry of M_yy (and the rhs terms) are
 * summed in one FIXED order (diagonal: a per-column warp tree; off-diagonal:
 * segmented shuffle trees over the plan's destination-sorted pair list), so the
 * result is bitwise reproducible; it differs from the elimination one sparse
 * variable at a time only by summation rounding.
 * Inputs (device): js_val[nnz] (values in the plan's CSR order); h_ss, sigma_s
 * [n_s]; H_dd [n_d x n_d, ldh, lower read]; sigma_d [n_d]; J_d [m x n_d, ldj];
 * d_h [m_I]; r [n_s + N] = (r_xs, r_xd, r_yg, r_yh) or NULL (then rhs_c is not
 * written).  Outputs (device): M [N x N, ldm, lower written], rhs_c [N] (or
 * NULL), w_out [n_s] (kept for mds_solve's recovery), anorm_out (one double,
 * or NULL: no norm).  work: device workspace of at least
 * mds_condense_workspace_size(plan, 1) bytes (per-entry products, norm
 * partials, the tile queue; no zeroing needed).
 * Data errors: MDS_ERR_NONPOSITIVE if some q_k <= 0 or d_h <= 0. */
size_t mds_condense_workspace_size(const mds_plan *plan, int64_t batch);
int mds_condense(const mds_plan *plan, const double *js_val, const double *h_ss, const double *sigma_s,
                 const double *H_dd, int64_t ldh, const double *sigma_d, const double *J_d, int64_t ldj,
                 const double *d_h, double delta_w, double delta_c, const double *r,
                 double *M, int64_t ldm, double *rhs_c, double *w_out, double *anorm_out,
                 int32_t *status_dev, void *work, size_t work_bytes, void *stream);

/* mds_condense_batched — the same for `batch` independent systems that share
 * the plan's sparsity pattern (SCOPF contingency scenarios, PAPER.md:70-78;
 * north star: "independent contingency KKT systems are batched per GPU").
 * Scenario s uses array X + s * str_X for every per-scenario array (strides in
 * ELEMENTS; H_dd / J_d / M keep their leading dimensions inside a scenario).
 * delta_w, delta_c: DEVICE arrays [batch] (NULL = 0).  status: device int32
 * [batch] (scenario s writes only status[s]; one failing scenario does not
 * affect the others).  anorm_out: device [batch] or NULL.  active: device int32
 * [batch] or NULL (all): scenarios with active[s] == 0 are left untouched (their M,
 * rhs_c, w, anorm, status keep their values) -- the inertia-correction loop
 * re-condenses only its failing scenarios.  One launch sequence for the whole
 * batch (tiles of all scenarios share one work queue).
 * work >= mds_condense_workspace_size(plan, batch). */
int mds_condense_batched(const mds_plan *plan, int64_t batch,
                         const double *js_val, int64_t str_val,
                         const double *h_ss, int64_t str_hss, const double *sigma_s, int64_t str_sig,
                         const double *H_dd, int64_t ldh, int64_t str_H,
                         const double *sigma_d, int64_t str_sd,
                         const double *J_d, int64_t ldj, int64_t str_J,
                         const double *d_h, int64_t str_dh,
                         const double *delta_w, const double *delta_c,
                         const double *r, int64_t str_r,
                         double *M, int64_t ldm, int64_t str_M,
                         double *rhs_c, int64_t str_rhs, double *w_out, int64_t str_w,
                         double *anorm_out, int32_t *status, const int32_t *active,
                         void *work, size_t work_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * mds_factor — Bunch-Kaufman LDL^T of the symmetric indefinite M (PAPER.md:191:
 * "MAGMA uses the Bunch-Kaufman diagonal pivoting method to form a LDL^T
 * factorization ... the inertia ... can be effectively computed from the D
 * matrix"), alpha = (1+sqrt(17))/8, blocked, FP64.
 * In place: on return M holds D and unit-L below the diagonal, in
 * EXPLICIT-permutation form  P M P^T = L D L^T.  A 2x2 block of D at (k,k+1)
 * keeps its diagonal entries on the diagonal and its off-diagonal d21 in the
 * UPPER slot (k, k+1) of M (the one upper-triangle element written), with
 * L(k+1,k) = 0.
 * piv [2N] (device int32, caller-owned): piv[0..N) = per-step pivot record in
 * LAPACK 1-based encoding (piv[k]=p+1 for a 1x1 pivot that interchanged k and
 * p; piv[k]=piv[k+1]=-(p+1) for a 2x2 pivot at (k,k+1)); piv[N..2N) = the
 * final permutation (row i of P M P^T is row piv[N+i] of M).  The pair (M,piv)
 * is consumed only by mds_solve.
 * zero_tol: pivots with |d| <= zero_tol count as zero; zero_tol < 0 selects
 * N * eps * ||M||_inf (reading R4 in DESIGN.md).
 * anorm: device pointer to ||M||_inf as written by mds_condense's anorm_out
 * (a NaN there means M is not finite -> MDS_ERR_NONFINITE), or NULL: then
 * mds_factor scans M itself first (one fixed-order pass over the lower
 * triangle, also detecting NaN/Inf).
 * inertia_dev: device mds_inertia (written).  inertia_host: if non-NULL the
 * call synchronises `stream` and copies the inertia there (3 integers cross
 * the bus, nothing else).
 * work: device workspace of at least mds_factor_workspace_size(N) bytes.
 * Data errors: MDS_ERR_NONFINITE if M holds NaN/Inf (then nothing is
 * factored). */
size_t mds_factor_workspace_size(int64_t N);
int mds_factor(int64_t N, double *M, int64_t ldm, int32_t *piv, double zero_tol,
               const double *anorm, mds_inertia *inertia_dev, mds_inertia *inertia_host, int32_t *status_dev,
               void *work, size_t work_bytes, void *stream);
/* mds_factor_batched — `batch` independent N x N factorizations (SCOPF scenario
 * batches; SURVEY §8(b) _batched) in ONE launch sequence: each
 * panel step is one launch for all scenarios (grid.y = scenario), and the DMMA
 * trailing update is one persistent launch whose tile queue spans every
 * scenario.  Scenario s: M + s * str_M (elements; 16-byte aligned M, even ldm
 * and str_M required: the update is TMA-fed), piv + s * str_piv (>= 2N),
 * inertia_dev[s], status[s] (device arrays [batch]); anorm: device [batch]
 * (mds_condense_batched's anorm_out) or NULL (each M is scanned).  One
 * non-finite scenario aborts only itself (status[s] = NONFINITE, identity
 * permutation).  active: device int32 [batch] or NULL (all); scenarios with
 * active[s] == 0 keep their factorization, piv, inertia and tolerance (requires
 * anorm != NULL).  Same factor format and pivot rule as mds_factor.  Never
 * synchronises.  work >= mds_factor_batched_workspace_size(N, batch). */
size_t mds_factor_batched_workspace_size(int64_t N, int64_t batch);
int mds_factor_batched(int64_t batch, int64_t N, double *M, int64_t ldm, int64_t str_M, int32_t *piv,
                       int64_t str_piv, double zero_tol, const double *anorm, mds_inertia *inertia_dev,
                       int32_t *status, const int32_t *active, void *work, size_t work_bytes, void *stream);
/* ||M||_inf and the zero-pivot tolerance the last mds_factor on `work` used
 * (host copies; synchronous).  For the parity tests of reading R4. */
int mds_factor_tol(const void *work, double *anorm_host, double *tol_host);
/* Counters of the last mds_factor on `work` (host copies; synchronous): out4 =
 * {panels, symmetric interchanges, columns decided by the exact BK steps (not
 * the speculative accepted prefix), 1 if aborted on non-finite input}. */
int mds_factor_stats(const void *work, int64_t *out4);

/* ---------------------------------------------------------------------------
 * mds_solve — x = P^T L^{-T} D^{-1} L^{-1} P rhs_c with mds_factor's output,
 * then the sparse-step recovery from the first block row of Eq.(5):
 *   dx_s = w .* (r_xs - J_s dy)        (K2 mixed sparse mat-vec)
 * Inputs (device): LD, piv from mds_factor; rhs_c [N]; js_val [nnz]; w [n_s]
 * (from mds_condense); r_xs [n_s].  Outputs (device): dxy [N] = (dx_d, dy_g,
 * dy_h); dx_s [n_s] (skipped if plan is NULL or dx_s is NULL).  dxy may alias
 * rhs_c.  work: >= mds_solve_workspace_size(N) bytes.
 * Data errors: MDS_ERR_SINGULAR if a 1x1 pivot has |d| <= zero_tol (same
 * meaning as in mds_factor; < 0 selects the value mds_factor computed, which it
 * leaves in its workspace — pass the same `fwork` pointer, or NULL to use 0). */
size_t mds_solve_workspace_size(int64_t N);
int mds_solve(const mds_plan *plan, int64_t N, const double *LD, int64_t ldm, const int32_t *piv,
              const double *rhs_c, const double *js_val, const double *w, const double *r_xs,
              double *dxy, double *dx_s, double zero_tol, const void *fwork,
              int32_t *status_dev, void *work, size_t work_bytes, void *stream);

/* mds_solve_batched — `batch` solves + recoveries with mds_factor_batched's
 * output in one launch sequence (grid.y = scenario).  Scenario s: LD + s * str_LD,
 * piv + s * str_piv, rhs_c + s * str_rhs, js_val + s * str_val, w + s * str_w,
 * r_xs + s * str_r, dxy + s * str_dxy, dx_s + s * str_dxs (elements), status[s];
 * fwork = the mds_factor_batched workspace (zero_tol < 0 reads scenario s's
 * tolerance from it).  work >= mds_solve_batched_workspace_size(N, batch). */
size_t mds_solve_batched_workspace_size(int64_t N, int64_t batch);
int mds_solve_batched(const mds_plan *plan, int64_t batch, int64_t N, const double *LD, int64_t ldm, int64_t str_LD,
                      const int32_t *piv, int64_t str_piv, const double *rhs_c, int64_t str_rhs,
                      const double *js_val, int64_t str_val, const double *w, int64_t str_w,
                      const double *r_xs, int64_t str_r, double *dxy, int64_t str_dxy, double *dx_s, int64_t str_dxs,
                      double zero_tol, const void *fwork, int32_t *status_dev, void *work, size_t work_bytes,
                      void *stream);

/* ---------------------------------------------------------------------------
 * ipm_step_vectors — barrier vector kernels (K1), one fused pass:
 * fraction-to-boundary ("the point that is feasible with respect
 * to the bounds constraints and is the farthest away ... requires a 'reduce'"),
 * complementarity and residual norms, optional barrier diagonal sigma.
 * Bounds with |b| >= 1e20 are infinite (reading R10).  tau in (0,1).
 *   out[0] alpha_p  = min(1, min tau*(x-lo)/(-dx) [dx<0], tau*(up-x)/dx [dx>0])
 *   out[1] alpha_d  = min(1, min tau*zl/(-dzl) [dzl<0], tau*zu/(-dzu) [dzu<0])
 *   out[2] compl_inf= max |(x-lo)*zl - mu|, |(up-x)*zu - mu|   (finite bounds)
 *   out[3] compl_sum= sum (x-lo)*zl + (up-x)*zu                (finite bounds)
 *   out[4] n_compl  = number of finite bounds (as double)
 *   out[5] first_bad= lowest index not strictly interior (or z<=0), else -1
 *   out[6+i] = ||res_i||_inf, i < n_res (n_res <= 8)
 * Inputs (device) x, dx, lo, up, zl, zu, dzl, dzu [n]; res: HOST array of
 * n_res device pointers, res_len: HOST array of their lengths.  Outputs
 * (device): out [6 + n_res] doubles; sigma_out [n] (= zl/(x-lo) + zu/(up-x),
 * infinite-bound terms 0) or NULL.  work: >= ipm_step_vectors_workspace_size(n)
 * bytes, ZEROED once before first use (the kernel leaves it zeroed).
 * Data errors: MDS_ERR_NOT_INTERIOR. */
size_t ipm_step_vectors_workspace_size(int64_t n);
/* ipm_step_vectors_batched — the same for `batch` scenarios in one launch: the 8
 * input vectors and sigma_out of scenario s at + s * str_vec (elements, >= n),
 * out + s * str_out (>= 6 + n_res), status[s]; tau / mu from the device arrays
 * tau_arr / mu_arr [batch] when non-NULL, else the scalars; residual j of
 * scenario s at res[j] + s * res_str[j] (res, res_len, res_str: HOST arrays).
 * work >= ipm_step_vectors_batched_workspace_size(n, batch) (no zeroing needed). */
size_t ipm_step_vectors_batched_workspace_size(int64_t n, int64_t batch);
int ipm_step_vectors_batched(int64_t batch, int64_t n, int64_t str_vec, const double *x, const double *dx,
                             const double *lo, const double *up, const double *zl, const double *zu,
                             const double *dzl, const double *dzu, double tau, double mu,
                             const double *tau_arr, const double *mu_arr, int32_t n_res,
                             const double *const *res, const int64_t *res_len, const int64_t *res_str,
                             double *out, int64_t str_out, double *sigma_out, int32_t *status_dev,
                             void *work, size_t work_bytes, void *stream);
int ipm_step_vectors(int64_t n, const double *x, const double *dx, const double *lo, const double *up,
                     const double *zl, const double *zu, const double *dzl, const double *dzu,
                     double tau, double mu, int32_t n_res, const double *const *res, const int64_t *res_len,
                     double *out, double *sigma_out, int32_t *status_dev,
                     void *work, size_t work_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * mds_kkt_residual — the K2 mixed sparse/dense mat-vec of PAPER.md:185 on the
 * FULL (uncondensed) Eq.(5) matrix of PAPER.md:147-159:
 *   K = [ Q_s     0      J_s  ]   Q_s = diag(h_ss + sigma_s + delta_w)
 *       [ 0       Q_d    J_d^T]   Q_d = H_dd + diag(sigma_d) + delta_w I
 *       [ J_s^T   J_d   -D_y  ]   D_y = diag(0_{m_E}, 1/d_h) + delta_c I
 * out = b - K x (b != NULL) or K x (b == NULL), x/b/out laid out
 * [x_s (n_s) | x_d (n_d) | y_g (m_E) | y_h (m_I)] (device, caller-owned, out
 * must not alias x).  The same inputs as mds_condense (same layouts, H_dd lower
 * read).  rnorm: optional device scalar, ||out||_inf.  work: >=
 * mds_kkt_residual_workspace_size(plan) bytes (per-tile partial sums: every
 * entry of the lower H_dd and of J_d is read once).  Used to check a whole Newton
 * step (condense + factor + solve + recovery) against the original system, and
 * as the residual of iterative refinement.  No data errors (argument errors
 * only); deterministic (fixed-order sums). */
size_t mds_kkt_residual_workspace_size(const mds_plan *plan);
int mds_kkt_residual(const mds_plan *plan, const double *js_val, const double *h_ss, const double *sigma_s,
                     const double *H_dd, int64_t ldh, const double *sigma_d, const double *J_d, int64_t ldj,
                     const double *d_h, double delta_w, double delta_c, const double *x, const double *b,
                     double *out, double *rnorm, void *work, size_t work_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * Inertia correction of a scenario batch on the device (
 * PAPER.md:161, 191; the multiples of the cited Algorithm IC, R22).
 * Per scenario a state machine advanced once per trial round by
 * mds_ic_step_batched from the trial's inertia and status: phase 0 = the (0,0)
 * trial was evaluated, 1 = a delta_w > 0 trial was evaluated, 2 = accepted,
 * 3 = failed (delta_w > delta_w_max: singular; the step writes MDS_ERR_SINGULAR
 * into status[s], so the solve and step vectors skip the scenario), 4 = data
 * error (status[s] already set by the trial).  active[s] = 1
 * exactly when scenario s needs another trial (delta_w[s], delta_c[s] set for
 * it); *any_active = OR over the batch.  The batched condense / factor take
 * `active` as their mask, so only failing scenarios are re-factored.  All
 * arrays are device [batch]; delta_w_last persists across Newton iterations
 * (warm start), the rest is reset by mds_ic_begin_batched (phase 0, active 1,
 * delta 0, ntrial 1).  mu: device [batch] or NULL (then the scalar).
 * mds_ic_graph_create captures the whole loop -- reset, first trial of every
 * scenario, step, then a CUDA-graph conditional WHILE node whose body is
 * (masked condense, masked factor, step) and whose condition the step kernel
 * sets with cudaGraphSetConditional -- into one graph; mds_ic_graph_launch runs
 * it on a stream: no host round trip per trial. */
typedef struct {
  double delta_w0, delta_w_min, delta_w_max, kappa_w_plus, kappa_w_plus_first, kappa_w_minus, delta_c_bar, kappa_c;
} mds_ic_params;
typedef struct {
  double *delta_w, *delta_c, *delta_w_last;
  int32_t *phase, *active, *ntrial, *any_active;
} mds_ic_state;
typedef struct {
  int64_t batch;
  const double *js_val; int64_t str_val;
  const double *h_ss; int64_t str_hss;
  const double *sigma_s; int64_t str_sig;
  const double *H_dd; int64_t ldh, str_H;
  const double *sigma_d; int64_t str_sd;
  const double *J_d; int64_t ldj, str_J;
  const double *d_h; int64_t str_dh;
  const double *r; int64_t str_r;
  double *M; int64_t ldm, str_M;
  double *rhs_c; int64_t str_rhs;
  double *w_out; int64_t str_w;
  double *anorm_out;
  int32_t *status;
  void *work; size_t work_bytes;
} mds_condense_batched_args;
typedef struct {
  int64_t batch, N;
  int32_t *piv; int64_t str_piv;
  double zero_tol;
  mds_inertia *inertia_dev;
  void *work; size_t work_bytes;
} mds_factor_batched_args;
typedef struct mds_ic_graph mds_ic_graph;
int mds_ic_begin_batched(int64_t batch, const mds_ic_state *st, void *stream);
int mds_ic_step_batched(int64_t batch, int64_t n_d, int64_t m, const mds_inertia *inertia, int32_t *status,
                        const double *mu_arr, double mu, const mds_ic_params *params, const mds_ic_state *st,
                        void *stream);
int mds_ic_graph_create(const mds_plan *plan, const mds_condense_batched_args *ca, const mds_factor_batched_args *fa,
                        int64_t n_d, int64_t m, const double *mu_arr, double mu, const mds_ic_params *params,
                        const mds_ic_state *st, mds_ic_graph **out);
int mds_ic_graph_launch(mds_ic_graph *graph, void *stream);
int mds_ic_graph_destroy(mds_ic_graph *graph);

/* ---------------------------------------------------------------------------
 * Interior-point loop vector kernels (K1 "axpy" + the filter line search's
 * reductions) for the convex-QP IPM of DESIGN.md R23.
 * One iterate: P = [x_s | x_d | s] (n + m_I; n = n_s + n_d), lo / up over P
 * (slack bounds h_l / h_u in the tail; |b| >= 1e20 infinite), bound duals zl / zu
 * over P (slack duals in the tail), y [m].  Kxy = (H x + J^T y, J x) is
 * mds_kkt_residual's K x with sigma = delta = 0 and d_h = +inf.  All device
 * pointers, caller-owned, stream-ordered, deterministic (fixed-order sums).
 *
 * ipm_rhs: sigma [n+m_I] = zl/(P-lo) + zu/(up-P) (finite terms; tail = D_h),
 *   r [n+m] = Eq.(5) right-hand side (r_x = -(Kxy_x + c - mu/(x-lo) + mu/(up-x)),
 *   r_yE = -(J_E x - g_E), r_yI = -(J_I x - s) + q/D_h), q [m_I] = y_h + mu/(s-h_l)
 *   - mu/(h_u-s), res_d [n+m_I] = stationarity (x: Kxy_x + c - zl + zu; s: -y_h
 *   - v_l + v_u), res_p [m] = (J_E x - g_E, J_I x - s).
 * ipm_directions: from the solve's (dx, dy) [n+m]: dP = (dx, ds), ds = (dy_h + q)/D_h,
 *   dzl = mu/gl - zl - (zl/gl) dP, dzu = mu/gu - zu + (zu/gu) dP, dx0[0..n) = dx.
 * ipm_reduce: mode 0 out[0..4) = ||res_d||_inf, ||res_p||_inf, max gap*z, max |gap*z - mu|;
 *   mode 1 out[0..6) = f, (H x + c).dx, dx.H dx, barrier part of grad(phi).dP,
 *   ||res_p||_1, sum log gaps (Kd = K0 (dx, 0)); mode 2 (trial alpha) out[0..2) =
 *   ||res_p + alpha (J dx - (0, ds))||_1, sum log gaps(P + alpha dP).
 *   work >= ipm_workspace_size(n, m_I) bytes, zeroed once before first use.
 * ipm_apply: P += alpha dP, y += alpha dy, z += alpha_d dz, then the dual safeguard
 *   z in [mu/(kappa_sigma gap), kappa_sigma mu/gap]; xy [n+m] = (x, y). */
size_t ipm_workspace_size(int64_t n, int64_t m_I);
int ipm_rhs(int64_t n, int64_t m_E, int64_t m_I, const double *Kxy, const double *c, const double *g_E,
            const double *P, const double *lo, const double *up, const double *zl, const double *zu,
            const double *y, double mu, double *sigma, double *r, double *q, double *res_d, double *res_p,
            void *stream);
int ipm_directions(int64_t n, int64_t m_E, int64_t m_I, const double *dxy, const double *q, const double *sigma,
                   const double *P, const double *lo, const double *up, const double *zl, const double *zu,
                   double mu, double *dP, double *dzl, double *dzu, double *dx0, void *stream);
int ipm_reduce(int mode, int64_t n, int64_t m_E, int64_t m_I, const double *P, const double *dP, const double *lo,
               const double *up, const double *zl, const double *zu, const double *y, const double *c,
               const double *Kxy, const double *Kd, const double *res_d, const double *res_p, double mu,
               double alpha, double *out, void *work, size_t work_bytes, void *stream);
int ipm_apply(int64_t n, int64_t m_E, int64_t m_I, double *P, double *zl, double *zu, double *y, double *xy,
              const double *dP, const double *dzl, const double *dzu, const double *dy, const double *lo,
              const double *up, double alpha, double alpha_d, double mu, double kappa_sigma, void *stream);

/* ---------------------------------------------------------------------------
 * Instrumentation (not on the hot path; used by bench.py for the roofline).
 * mds_launch_count: number of kernels this library has launched since load.
 * mds_profile_begin / mds_profile_end: while enabled, every kernel launch of
 * the four calls above is bracketed by CUDA events recorded on its own stream;
 * mds_profile_end synchronises those events and returns, per kernel class
 * (MDS_PROF_* below, ncls >= MDS_PROF_COUNT), the summed duration in ms and
 * the launch count.  Never enable while capturing a CUDA graph.
 * mds_factor_panels: after mds_factor, copies the first column of every panel
 * into starts_host[cap] (synchronous) and returns the number of panels, so
 * the caller can compute the trailing update's algorithmic flops exactly. */
enum {
    MDS_PROF_CONDENSE_W = 0, MDS_PROF_CONDENSE_DENSE, MDS_PROF_CONDENSE_YY, MDS_PROF_ANORM,
    MDS_PROF_PANEL_DIAG, MDS_PROF_PANEL_TRSM, MDS_PROF_PANEL_STORE, MDS_PROF_PANEL_SLOW, MDS_PROF_UPDATE,
    MDS_PROF_FINALIZE, MDS_PROF_SOLVE_GATHER, MDS_PROF_SOLVE_FWD, MDS_PROF_SOLVE_D, MDS_PROF_SOLVE_BWD,
    MDS_PROF_SOLVE_SCATTER, MDS_PROF_RECOVER, MDS_PROF_VECTORS, MDS_PROF_COUNT
};
unsigned long long mds_launch_count(void);
/* Tuning knob (process-wide): cap the CTA count of mds_factor's persistent
 * trailing-update kernels and of the multi-CTA exact-pivot panel (0 = one per
 * SM, the default).  Used when several factorizations run concurrently on
 * different streams (SCOPF batches).  A cap below the SM count also selects
 * the concurrent launch structure (no one-launch tail panels, whose waiting
 * CTAs would hold SMs other streams need); results are bitwise identical for
 * every cap value below the SM count, and differ from the uncapped structure
 * only by rounding order. */
int mds_factor_set_grid_cap(int ctas);
/* Launch-structure variants of mds_factor / mds_solve for A/B measurement and
 * for the variant parity tests (process-wide; the library never reads the
 * environment).  Every variant computes the same Bunch-Kaufman factorization
 * (same pivot rule, same inertia); results differ only by rounding order.
 * key: "default" (reset all), "tail_rows" (panels with at most this many rows
 * left use the one-launch tail path; < 0 = built-in choice), "exact_rows"
 * (rows per CTA of the multi-CTA exact panel, >= 32), and the flags "no_tma",
 * "no_lookahead", "static_sched", "no_snake", "no_cprefetch", "upd_inplace",
 * "upd_main", "slow_1cta", "exact_no_ls", "f2_trsm", "no_pdl", "ozaki",
 * "exact_cluster" (value 0/1; exact_cluster: the exact panel runs as one
 * thread-block cluster when it fits -- faster on pivot-heavy matrices, slower
 * by ~0.4 us per panel when every panel takes the fast path);
 * for mds_condense[_batched]: "cdense_ctas" (1..8), "cdense_serial",
 * "cdense_tma" (0/1) and "cond_group" (batched pair tiles: scenarios whose
 * tiles are interleaved in the work order, 1..65536; bitwise identical results
 * for every value -- each tile's sums do not depend on the order).
 * Returns MDS_ERR_ARG for an unknown key.  Not thread-safe against concurrent
 * mds_factor calls (set it between calls). */
int mds_set_variant(const char *key, long long value);
int mds_profile_begin(void);
int mds_profile_end(double *ms_by_class, int64_t *launches_by_class, int ncls);
int64_t mds_factor_panels(const void *fwork, int64_t N, int32_t *starts_host, int64_t cap);
/* Per-launch timeline of the last mds_profile_begin/end region: out3[3*i..] =
 * (class, start_ms, end_ms) relative to the first profiled launch; returns the
 * number of launches (copies at most cap). */
int64_t mds_profile_timeline(double *out3, int64_t cap);

/* ---------------------------------------------------------------------------
 * Distributed LDL^T of ONE system across GPUs (the paper's
 * implementation is single-GPU, larger systems future work,
 * PAPER.md:100).  One process per GPU; the lower triangle of M is cut into
 * 64-column panels, panel g owned by rank g mod P (1-D block-cyclic), each rank
 * storing its panels full height (column-major, global row index, ld >= N).
 * paper_2605_13736_b200/dist.py runs the panel loop and the collectives
 * (torch.distributed); these calls are its device work, all stream-ordered,
 * device pointers, argument errors returned, no data-dependent status.
 *
 * mds_dist_panel — on the panel's owner: the speculative (unpivoted) LDL^T of
 *   the n x nb panel A (rows k0..N-1 of its columns, lda): L (unit lower; may
 *   alias A with ldl == lda), W = L D (the columns at elimination), d[nb],
 *   cmax[nb] (in-block column maxima), parts (workspace, >= ceil((n-nb)/128) x 64
 *   doubles, nparts_cap = its rows), and the Bunch-Kaufman 1x1 acceptance test
 *   |d_j| >= alpha max_i |W(i, j)| for every column (alpha =
 *   (1+sqrt 17)/8): *accepted = 1 and inertia[0..2] += the counts of D (zero
 *   band |d| <= tol), else *accepted = 0 (the caller then factors the Schur
 *   complement from this panel on with mds_factor; inertia adds, Haynsworth).
 * mds_dist_update — C -= L W^T on nq local panels (global first column kq[q],
 *   width wq[q], stored at C + q*64*ldc; rows i >= kq[q]); L, W: rows k0..N-1 of
 *   the broadcast panel (ldl); max_rows = N - min(kq).  FP64 DMMA.
 * mds_dist_trsv64 — y := L11^-1 y (mode 0) or L11^-T y (mode 1), L11 unit lower nb x nb.
 * mds_dist_gemv_n — acc[i] += sum_t L(i, t) y[t], rows r0 <= i < r1 (global row index).
 * mds_dist_gemv_t — out[t] = sum_{r0 <= i < r1} L(i, t) x[i], t < nb.
 * mds_dist_rowabs — rs[i] = this rank's share of the row abs-sum of symmetric M
 *   (lower stored) for ||M||_inf: sum over its columns c <= i of |M(i, c)| plus,
 *   for its column i, sum_{r > i} |M(r, i)|; fixed order.  Sum rs over ranks. */
int mds_dist_panel(int64_t n, int nb, const double *A, int64_t lda, double *L, double *W, int64_t ldl, double *d,
                   double *cmax, double *parts, int64_t nparts_cap, double tol, int32_t *accepted,
                   long long *inertia, void *stream);
int mds_dist_update(int64_t N, int64_t k0, int nb, const double *L, const double *W, int64_t ldl, double *C,
                    int64_t ldc, const int64_t *kq, const int *wq, int nq, int64_t max_rows, void *stream);
int mds_dist_trsv64(int nb, const double *L, int64_t ldl, double *y, int mode, void *stream);
int mds_dist_gemv_n(int64_t r0, int64_t r1, int nb, const double *L, int64_t ldl, const double *y, double *acc,
                    void *stream);
int mds_dist_gemv_t(int64_t r0, int64_t r1, int nb, const double *L, int64_t ldl, const double *x, double *out,
                    void *stream);
int mds_dist_rowabs(int64_t N, const double *C, int64_t ldc, const int64_t *kq, const int *wq, int nq, double *rs,
                    void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MDS_B200_H */
