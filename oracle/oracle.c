/*
 * oracle.c — TEST INFRASTRUCTURE ONLY. Plain, slow, obviously-correct CPU
 * reference of the condensed-KKT hot path of the mixed dense-sparse (MDS)
 * interior-point method of arxiv/paper_2605_13736 (§2, Eq.(5)-(6)).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2605_13736_b200/) never does: it shares no code, headers, tables or
 * helpers with this file.
 *
 * Conventions:
 *   - FP64 throughout, compiled with -O2 -ffp-contract=off (no FMA contraction).
 *   - Dense symmetric matrices: column-major, leading dimension ld, LOWER
 *     triangle referenced (LAPACK uplo='L'); element (i,j), i>=j, at A[i + j*ld].
 *   - J_s is CSR n_s x m, ROWS = sparse variables (the north star
 *     writes J_s^T D J_s); column c < m_E is an equality (g) row of Eq.(5),
 *     c >= m_E an inequality (h) row.
 *   - Unknown ordering of M is (x_d, y_g, y_h) as Eq.(6).
 *
 * Parity status of each function is stated in DESIGN.md §Oracle pins; every
 * function here is pinned by a "not gpu" test in tests/test_oracle_*.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Threads the factorization's column loop may use (OpenMP; 1 without it).
 * Results are bit-identical for every thread count. */
int or_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void or_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

#define OR_OK 0
#define OR_ERR_ARG (-1)
#define OR_ERR_PATTERN (-2)
#define OR_ERR_NONPOSITIVE (-3)
#define OR_ERR_NONFINITE (-4)
#define OR_ERR_SINGULAR (-5)
#define OR_ERR_NOT_INTERIOR (-6)

#define AT(A, ld, i, j) ((A)[(size_t)(i) + (size_t)(j) * (size_t)(ld)])

/* ------------------------------------------------------------------------
 * O1. Condensation: Eq.(5) -> Eq.(6) by Gauss elimination of the sparse
 * block ("we use a Gauss elimination of the sparse blocks").
 *
 *   q_k = h_ss[k] + sigma_s[k] + delta_w      (Q_{x_s} = diag Hessian + D_{x_s},
 *                                             PAPER.md:159; +delta_w)
 *   w_k = 1 / q_k                              (Q_{x_s}^{-1}, assumption A2 PAPER.md:121)
 *   M_xx = H_dd + diag(sigma_d) + delta_w I    (Q_{x_d}, block (1,1) of Eq.(6))
 *   M_yx = J_d                                 (blocks (2,1),(3,1) of Eq.(6))
 *   M_yy = -J_s^T diag(w) J_s - diag(0_{m_E}, 1/d_h) - delta_c I
 *                                              (blocks (2,2),(2,3),(3,3) of Eq.(6);
 *                                               -delta_c I)
 *   rhs_c = [ r_xd ; r_y - J_s^T (w .* r_xs) ] (block elimination of Eq.(5), reading R12)
 *
 * r is [r_xs (n_s) ; r_xd (n_d) ; r_yg (m_E) ; r_yh (m_I)] as in Eq.(5).
 * Only the lower triangle of M is written.  Returns OR_ERR_NONPOSITIVE if some
 * q_k <= 0 or d_h <= 0, OR_ERR_PATTERN for a non-canonical CSR.
 * ------------------------------------------------------------------------ */
int or_condense(int64_t n_s, int64_t n_d, int64_t m_E, int64_t m_I,
                const int32_t *rowptr, const int32_t *colidx, const double *val,
                const double *h_ss, const double *sigma_s,
                const double *H_dd, int64_t ldh, const double *sigma_d,
                const double *J_d, int64_t ldj, const double *d_h,
                double delta_w, double delta_c, const double *r,
                double *M, int64_t ldm, double *rhs_c, double *w_out)
{
    int64_t m = m_E + m_I, N = n_d + m;
    if (n_s < 0 || n_d < 0 || m_E < 0 || m_I < 0 || ldm < (N > 0 ? N : 1)) return OR_ERR_ARG;
    /* CSR must be canonical: sorted, unique, in range (reading R13) */
    if (rowptr[0] != 0) return OR_ERR_PATTERN;
    for (int64_t k = 0; k < n_s; k++) {
        if (rowptr[k + 1] < rowptr[k]) return OR_ERR_PATTERN;
        for (int64_t p = rowptr[k]; p < rowptr[k + 1]; p++) {
            if (colidx[p] < 0 || colidx[p] >= m) return OR_ERR_PATTERN;
            if (p > rowptr[k] && colidx[p] <= colidx[p - 1]) return OR_ERR_PATTERN;
        }
    }
    for (int64_t i = 0; i < m_I; i++)
        if (!(d_h[i] > 0.0)) return OR_ERR_NONPOSITIVE;

    /* step 1: block (1,1) = Q_{x_d} = H_dd + diag(sigma_d) + delta_w I */
    for (int64_t j = 0; j < n_d; j++)
        for (int64_t i = j; i < n_d; i++) {
            double v = AT(H_dd, ldh, i, j);
            if (i == j) v = v + sigma_d[j] + delta_w;
            AT(M, ldm, i, j) = v;
        }
    /* step 2: blocks (2,1),(3,1) = J_d (the lower triangle holds J_d, not J_d^T) */
    for (int64_t j = 0; j < n_d; j++)
        for (int64_t c = 0; c < m; c++)
            AT(M, ldm, n_d + c, j) = AT(J_d, ldj, c, j);
    /* step 3: block (2:3,2:3) starts at -diag(0, 1/d_h) - delta_c I */
    for (int64_t c2 = 0; c2 < m; c2++)
        for (int64_t c1 = c2; c1 < m; c1++) {
            double v = 0.0;
            if (c1 == c2) {
                v = -delta_c;
                if (c1 >= m_E) v = v - 1.0 / d_h[c1 - m_E];
            }
            AT(M, ldm, n_d + c1, n_d + c2) = v;
        }
    /* step 4: M_yy -= J_s^T diag(w) J_s, one sparse variable at a time */
    for (int64_t k = 0; k < n_s; k++) {
        double q = h_ss[k] + sigma_s[k] + delta_w;
        if (!(q > 0.0)) return OR_ERR_NONPOSITIVE;
        double w = 1.0 / q;
        if (w_out) w_out[k] = w;
        for (int64_t p = rowptr[k]; p < rowptr[k + 1]; p++) {
            double t = val[p] * w;
            for (int64_t pp = rowptr[k]; pp <= p; pp++) {
                /* colidx sorted: colidx[p] >= colidx[pp] -> lower triangle */
                AT(M, ldm, n_d + colidx[p], n_d + colidx[pp]) -= t * val[pp];
            }
        }
    }
    /* step 5: rhs_c */
    if (rhs_c && r) {
        for (int64_t j = 0; j < n_d; j++) rhs_c[j] = r[n_s + j];
        for (int64_t c = 0; c < m; c++) rhs_c[n_d + c] = r[n_s + n_d + c];
        for (int64_t k = 0; k < n_s; k++) {
            double w = 1.0 / (h_ss[k] + sigma_s[k] + delta_w);
            double wr = w * r[k];
            for (int64_t p = rowptr[k]; p < rowptr[k + 1]; p++)
                rhs_c[n_d + colidx[p]] -= val[p] * wr;
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------
 * ||A||_inf of a symmetric matrix from its lower triangle (row abs-sums using
 * symmetry).  Also detects non-finite entries (reading R17).
 * Used for the zero-pivot tolerance tol = N * eps * ||A||_inf (reading R4).
 * ------------------------------------------------------------------------ */
int or_anorm_lower(int64_t N, const double *A, int64_t lda, double *anorm)
{
    double best = 0.0;
    for (int64_t i = 0; i < N; i++) {
        double s = 0.0;
        for (int64_t j = 0; j <= i; j++) {
            double v = AT(A, lda, i, j);
            if (!isfinite(v)) return OR_ERR_NONFINITE;
            s += fabs(v);
        }
        for (int64_t j = i + 1; j < N; j++) s += fabs(AT(A, lda, j, i));
        if (s > best) best = s;
    }
    *anorm = best;
    return OR_OK;
}

/* ------------------------------------------------------------------------
 * O2. Unpivoted LDL^T (reference for SPD / quasi-definite inputs, which the
 * G1 generator produces).  In place: D on the diagonal, unit-L below.
 * Fails (OR_ERR_SINGULAR) if some |d_k| <= tol.
 * ------------------------------------------------------------------------ */
int or_ldlt_nopiv(int64_t N, double *A, int64_t lda, double tol)
{
    for (int64_t k = 0; k < N; k++) {
        double d = AT(A, lda, k, k);
        if (!(fabs(d) > tol)) return OR_ERR_SINGULAR;
        /* A22 -= a a^T / d (lower), with a = A[k+1:,k] unscaled */
        for (int64_t j = k + 1; j < N; j++) {
            double t = AT(A, lda, j, k) / d;
            for (int64_t i = j; i < N; i++)
                AT(A, lda, i, j) -= AT(A, lda, i, k) * t;
        }
        for (int64_t i = k + 1; i < N; i++) AT(A, lda, i, k) /= d;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------
 * O3. Bunch-Kaufman LDL^T, LAPACK dsytf2 uplo='L' semantics (the method the
 * paper's solver uses: "MAGMA uses the Bunch-Kaufman diagonal pivoting method
 * to form a LDL^T factorization").  alpha = (1+sqrt(17))/8
 * (reading R6); argmax = first index attaining the maximum (reading R5).
 * Output: A overwritten with D (diagonal, plus subdiagonal for 2x2 blocks) and
 * the multipliers of L below it in LAPACK product form (already-factored
 * columns are NOT row-swapped); ipiv in LAPACK 1-based encoding:
 *   ipiv[k] = p+1  (1x1 pivot, rows/cols k and p interchanged),
 *   ipiv[k] = ipiv[k+1] = -(p+1) (2x2 pivot, rows/cols k+1 and p interchanged).
 * Returns info: 0, or k+1 for the first exactly-zero pivot column.
 * ------------------------------------------------------------------------ */
static int64_t or_iamax(int64_t n, const double *x, int64_t inc)
{
    /* first index of max |x_i| (BLAS IDAMAX semantics, 0-based) */
    int64_t best = 0;
    double bv = -1.0;
    for (int64_t i = 0; i < n; i++) {
        double v = fabs(x[i * inc]);
        if (v > bv) { bv = v; best = i; }
    }
    return best;
}

int64_t or_bk_factor(int64_t N, double *A, int64_t lda, int32_t *ipiv)
{
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    int64_t info = 0;
    int64_t k = 0;
    while (k < N) {
        int kstep = 1;
        int64_t kp;
        double absakk = fabs(AT(A, lda, k, k));
        int64_t imax = k;
        double colmax = 0.0;
        if (k < N - 1) {
            imax = k + 1 + or_iamax(N - k - 1, &AT(A, lda, k + 1, k), 1);
            colmax = fabs(AT(A, lda, imax, k));
        }
        if (absakk == 0.0 && colmax == 0.0) {
            /* column k is exactly zero: zero pivot, nothing to eliminate */
            if (info == 0) info = k + 1;
            kp = k;
            ipiv[k] = (int32_t)(k + 1);
            k += 1;
            continue;
        }
        if (absakk >= alpha * colmax) {
            kp = k;
        } else {
            /* rowmax = largest off-diagonal magnitude in row/column imax */
            int64_t jmax = k + or_iamax(imax - k, &AT(A, lda, imax, k), lda);
            double rowmax = fabs(AT(A, lda, imax, jmax));
            if (imax < N - 1) {
                jmax = imax + 1 + or_iamax(N - imax - 1, &AT(A, lda, imax + 1, imax), 1);
                double v = fabs(AT(A, lda, jmax, imax));
                if (v > rowmax) rowmax = v;
            }
            if (absakk >= alpha * colmax * (colmax / rowmax)) {
                kp = k;
            } else if (fabs(AT(A, lda, imax, imax)) >= alpha * rowmax) {
                kp = imax;
            } else {
                kp = imax;
                kstep = 2;
            }
        }
        int64_t kk = k + kstep - 1;
        if (kp != kk) {
            /* symmetric interchange of rows/cols kk and kp in the trailing
               submatrix A(kk:N, kk:N) only (LAPACK product form) */
            for (int64_t i = kp + 1; i < N; i++) {
                double t = AT(A, lda, i, kk); AT(A, lda, i, kk) = AT(A, lda, i, kp); AT(A, lda, i, kp) = t;
            }
            for (int64_t j = kk + 1; j < kp; j++) {
                double t = AT(A, lda, j, kk); AT(A, lda, j, kk) = AT(A, lda, kp, j); AT(A, lda, kp, j) = t;
            }
            { double t = AT(A, lda, kk, kk); AT(A, lda, kk, kk) = AT(A, lda, kp, kp); AT(A, lda, kp, kp) = t; }
            if (kstep == 2) {
                double t = AT(A, lda, k + 1, k); AT(A, lda, k + 1, k) = AT(A, lda, kp, k); AT(A, lda, kp, k) = t;
            }
        }
        if (kstep == 1) {
            /* 1x1: A22 -= (1/d) a a^T ; a /= d   (dsyr + dscal) */
            double r1 = 1.0 / AT(A, lda, k, k);
            /* columns j are independent (each keeps its own serial update
               sequence), so the OpenMP split is bit-identical to 1 thread */
            #pragma omp parallel for schedule(static) if (N - k > 512)
            for (int64_t j = k + 1; j < N; j++) {
                double temp = -r1 * AT(A, lda, j, k);
                for (int64_t i = j; i < N; i++)
                    AT(A, lda, i, j) = AT(A, lda, i, j) + AT(A, lda, i, k) * temp;
            }
            for (int64_t i = k + 1; i < N; i++) AT(A, lda, i, k) = r1 * AT(A, lda, i, k);
            ipiv[k] = (int32_t)(kp + 1);
        } else {
            /* 2x2: LAPACK dsytf2 scaled formulas */
            if (k < N - 2) {
                double d21 = AT(A, lda, k + 1, k);
                double d11 = AT(A, lda, k + 1, k + 1) / d21;
                double d22 = AT(A, lda, k, k) / d21;
                double t = 1.0 / (d11 * d22 - 1.0);
                d21 = t / d21;
                /* dsytf2's loop computes (wk, wkp1) of column j from the ORIGINAL
                   A(j,k), A(j,k+1), updates A(j:,j) with the original A(j:,k),
                   A(j:,k+1), then stores (wk, wkp1) into A(j,k), A(j,k+1).  The
                   three steps are done here as three passes so the column update
                   can be split over threads: same operations, same operands,
                   bit-identical to the serial loop. */
                double *wk = (double *)malloc(sizeof(double) * 2 * (size_t)N);
                double *wkp1 = wk + N;
                for (int64_t j = k + 2; j < N; j++) {
                    wk[j] = d21 * (d11 * AT(A, lda, j, k) - AT(A, lda, j, k + 1));
                    wkp1[j] = d21 * (d22 * AT(A, lda, j, k + 1) - AT(A, lda, j, k));
                }
                #pragma omp parallel for schedule(static) if (N - k > 512)
                for (int64_t j = k + 2; j < N; j++) {
                    for (int64_t i = j; i < N; i++)
                        AT(A, lda, i, j) = AT(A, lda, i, j) - AT(A, lda, i, k) * wk[j] - AT(A, lda, i, k + 1) * wkp1[j];
                }
                for (int64_t j = k + 2; j < N; j++) {
                    AT(A, lda, j, k) = wk[j];
                    AT(A, lda, j, k + 1) = wkp1[j];
                }
                free(wk);
            }
            ipiv[k] = (int32_t)(-(kp + 1));
            ipiv[k + 1] = (int32_t)(-(kp + 1));
        }
        k += kstep;
    }
    return info;
}

/* ------------------------------------------------------------------------
 * O4. Inertia from the block-diagonal D ("the inertia ... can be
 * effectively computed from the D matrix (which is block diagonal with blocks
 * of size 1x1 and 2x2 pivots)").  1x1 pivot d: pos if d > tol, neg if
 * d < -tol, zero otherwise.  2x2 block: (1,0,1) — BK's test guarantees
 * det < 0; the oracle asserts it (returns OR_ERR_ARG if violated).
 * out = {pos, zero, neg}.
 * ------------------------------------------------------------------------ */
int or_inertia(int64_t N, const double *A, int64_t lda, const int32_t *ipiv, double tol, int64_t *out)
{
    int64_t pos = 0, zero = 0, neg = 0;
    int64_t k = 0;
    while (k < N) {
        if (ipiv[k] > 0) {
            double d = AT(A, lda, k, k);
            if (d > tol) pos++;
            else if (d < -tol) neg++;
            else zero++;
            k += 1;
        } else {
            double a = AT(A, lda, k, k), b = AT(A, lda, k + 1, k), c = AT(A, lda, k + 1, k + 1);
            double det = a * c - b * b;
            if (!(det < 0.0)) return OR_ERR_ARG;
            pos++; neg++;
            k += 2;
        }
    }
    out[0] = pos; out[1] = zero; out[2] = neg;
    return OR_OK;
}

/* ------------------------------------------------------------------------
 * O5. Solve with the BK factors, LAPACK dsytrs uplo='L' semantics:
 * x = P L^{-T} D^{-1} L^{-1} P^T b, in place in b.  A zero 1x1 pivot
 * (|d| <= tol) gives OR_ERR_SINGULAR (reading R4).
 * ------------------------------------------------------------------------ */
int or_bk_solve(int64_t N, const double *A, int64_t lda, const int32_t *ipiv, double *b, double tol)
{
    int64_t k = 0;
    while (k < N) { /* forward: L D y = P^T b */
        if (ipiv[k] > 0) {
            int64_t kp = ipiv[k] - 1;
            if (kp != k) { double t = b[k]; b[k] = b[kp]; b[kp] = t; }
            for (int64_t i = k + 1; i < N; i++) b[i] -= AT(A, lda, i, k) * b[k];
            double d = AT(A, lda, k, k);
            if (!(fabs(d) > tol)) return OR_ERR_SINGULAR;
            b[k] /= d;
            k += 1;
        } else {
            int64_t kp = -ipiv[k] - 1;
            if (kp != k + 1) { double t = b[k + 1]; b[k + 1] = b[kp]; b[kp] = t; }
            for (int64_t i = k + 2; i < N; i++) b[i] -= AT(A, lda, i, k) * b[k];
            for (int64_t i = k + 2; i < N; i++) b[i] -= AT(A, lda, i, k + 1) * b[k + 1];
            double akm1k = AT(A, lda, k + 1, k);
            double akm1 = AT(A, lda, k, k) / akm1k;
            double ak = AT(A, lda, k + 1, k + 1) / akm1k;
            double denom = akm1 * ak - 1.0;
            double bkm1 = b[k] / akm1k;
            double bk = b[k + 1] / akm1k;
            b[k] = (ak * bkm1 - bk) / denom;
            b[k + 1] = (akm1 * bk - bkm1) / denom;
            k += 2;
        }
    }
    k = N - 1;
    while (k >= 0) { /* backward: L^T x = y, then undo P */
        if (ipiv[k] > 0) {
            double s = 0.0;
            for (int64_t i = k + 1; i < N; i++) s += AT(A, lda, i, k) * b[i];
            b[k] -= s;
            int64_t kp = ipiv[k] - 1;
            if (kp != k) { double t = b[k]; b[k] = b[kp]; b[kp] = t; }
            k -= 1;
        } else {
            double s = 0.0, s1 = 0.0;
            for (int64_t i = k + 1; i < N; i++) s += AT(A, lda, i, k) * b[i];
            for (int64_t i = k + 1; i < N; i++) s1 += AT(A, lda, i, k - 1) * b[i];
            b[k] -= s;
            b[k - 1] -= s1;
            int64_t kp = -ipiv[k] - 1;
            if (kp != k) { double t = b[k]; b[k] = b[kp]; b[kp] = t; }
            k -= 2;
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------
 * O6. Sparse-step recovery (back-substitution of the eliminated block of
 * Eq.(5), first block row): Q_{x_s} dx_s + J_s dy = r_xs
 *   => dx_s = w .* (r_xs - J_s dy)      (K2 mixed sparse mat-vec)
 * dy = (dy_g, dy_h), length m.
 * ------------------------------------------------------------------------ */
void or_recover(int64_t n_s, const int32_t *rowptr, const int32_t *colidx, const double *val,
                const double *w, const double *r_xs, const double *dy, double *dx_s)
{
    for (int64_t k = 0; k < n_s; k++) {
        double s = 0.0;
        for (int64_t p = rowptr[k]; p < rowptr[k + 1]; p++) s += val[p] * dy[colidx[p]];
        dx_s[k] = w[k] * (r_xs[k] - s);
    }
}

/* ------------------------------------------------------------------------
 * O7. Barrier vector kernels (K1; fraction-to-boundary
 * "farthest feasible point along the direction").
 * Bounds with |b| >= 1e20 are infinite (reading R10).
 *   alpha_p = min(1, min_{lo finite, dx<0} tau*(x-lo)/(-dx), min_{up finite, dx>0} tau*(up-x)/dx)
 *   alpha_d = min(1, min_{lo finite, dzl<0} tau*zl/(-dzl), min_{up finite, dzu<0} tau*zu/(-dzu))
 *   compl_inf = max over finite bounds of |(x-lo)*zl - mu|, |(up-x)*zu - mu|
 *   compl_sum = sum over finite bounds of (x-lo)*zl + (up-x)*zu ; n_compl = count
 *   sigma[i]  = zl/(x-lo) + zu/(up-x) (infinite-bound terms 0)   (D_x)
 * NOT_INTERIOR if x is not strictly inside a finite bound or the bound dual
 * is not > 0; first_bad = lowest such index.
 * out: [alpha_p, alpha_d, compl_inf, compl_sum, n_compl, first_bad]
 * ------------------------------------------------------------------------ */
int or_step_vectors(int64_t n, const double *x, const double *dx, const double *lo, const double *up,
                    const double *zl, const double *zu, const double *dzl, const double *dzu,
                    double tau, double mu, double *out, double *sigma)
{
    const double INF = 1e20;
    double ap = 1.0, ad = 1.0, cinf = 0.0, csum = 0.0;
    int64_t nc = 0, bad = -1;
    for (int64_t i = 0; i < n; i++) {
        int hl = fabs(lo[i]) < INF, hu = fabs(up[i]) < INF;
        double s = 0.0;
        if (hl) {
            double gap = x[i] - lo[i];
            if (!(gap > 0.0) || !(zl[i] > 0.0)) { if (bad < 0) bad = i; }
            if (dx[i] < 0.0) { double a = tau * gap / (-dx[i]); if (a < ap) ap = a; }
            if (dzl[i] < 0.0) { double a = tau * zl[i] / (-dzl[i]); if (a < ad) ad = a; }
            double c = gap * zl[i];
            double e = fabs(c - mu);
            if (e > cinf) cinf = e;
            csum += c; nc++;
            s += zl[i] / gap;
        }
        if (hu) {
            double gap = up[i] - x[i];
            if (!(gap > 0.0) || !(zu[i] > 0.0)) { if (bad < 0) bad = i; }
            if (dx[i] > 0.0) { double a = tau * gap / dx[i]; if (a < ap) ap = a; }
            if (dzu[i] < 0.0) { double a = tau * zu[i] / (-dzu[i]); if (a < ad) ad = a; }
            double c = gap * zu[i];
            double e = fabs(c - mu);
            if (e > cinf) cinf = e;
            csum += c; nc++;
            s += zu[i] / gap;
        }
        if (sigma) sigma[i] = s;
    }
    out[0] = ap; out[1] = ad; out[2] = cinf; out[3] = csum; out[4] = (double)nc; out[5] = (double)bad;
    return bad >= 0 ? OR_ERR_NOT_INTERIOR : OR_OK;
}

/* ||v||_inf of a residual vector (K1 "computing residual norms") */
double or_norm_inf(int64_t n, const double *v)
{
    double b = 0.0;
    for (int64_t i = 0; i < n; i++) { double a = fabs(v[i]); if (a > b) b = a; }
    return b;
}
