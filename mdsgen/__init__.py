"""Seeded synthetic input generators for the condensed-KKT hot path.

This module is shared by the CPU oracle's tests and the CUDA path's tests and
benchmark.  It holds NONE of the method's arithmetic (no condensation, no
factorization, no solve): it only draws inputs with the shapes, sparsity and
value distributions of the paper's workloads (DESIGN.md §Input recipe;
SURVEY.md §8(d) generators G1-G5).

Conventions: J_s is CSR n_s x m with rows = sparse variables (reading R1);
dense matrices are numpy Fortran-order (column-major) arrays; bounds with
|b| >= 1e20 are infinite (reading R10).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

INF = 1e20

# BASELINE.json configs -> concrete shapes (readings in DESIGN.md)
CONFIGS = {
    "C1": dict(n_s=400, n_d=20, m_E=10, m_I=10),
    "C2": dict(n_s=100_000, n_d=512, m_E=256, m_I=256),
    "C3": dict(n_s=1_000_000, n_d=4096, m_E=2048, m_I=2048),
    "C4": dict(n_s=131_072, n_d=1024, m_E=512, m_I=512),
}


@dataclass
class MDSProblem:
    """Inputs of one Newton step's KKT system, Eq.(5) of PAPER.md:147-159."""
    n_s: int
    n_d: int
    m_E: int
    m_I: int
    rowptr: np.ndarray          # int32[n_s+1]
    colidx: np.ndarray          # int32[nnz], sorted & unique per row
    val: np.ndarray             # f64[nnz]
    h_ss: np.ndarray            # f64[n_s]  diag of Hessian of L in x_s (A2: >= 0)
    sigma_s: np.ndarray         # f64[n_s]  D_{x_s}
    H_dd: np.ndarray            # f64[n_d, n_d] Fortran, symmetric (lower referenced)
    sigma_d: np.ndarray         # f64[n_d]  D_{x_d}
    J_d: np.ndarray             # f64[m, n_d] Fortran
    d_h: np.ndarray             # f64[m_I]  D_h > 0
    delta_w: float = 0.0
    delta_c: float = 0.0
    r: Optional[np.ndarray] = None   # f64[n_s + n_d + m]: (r_xs, r_xd, r_yg, r_yh)
    expected_inertia: Optional[tuple] = None   # closed-form inertia of M when known
    meta: dict = field(default_factory=dict)

    @property
    def m(self):
        return self.m_E + self.m_I

    @property
    def N(self):
        return self.n_d + self.m_E + self.m_I

    @property
    def nnz(self):
        return int(self.rowptr[-1])


def _distinct_rows(rng, n_rows, k, m, pattern, window=64):
    """n_rows x k int matrix of distinct constraint indices per row, sorted."""
    k = min(k, m)
    if n_rows == 0 or k == 0:
        return np.zeros((n_rows, k), dtype=np.int64)
    if pattern == "uniform":
        idx = rng.integers(0, m, size=(n_rows, k))
    elif pattern == "local":
        w = min(window, m)
        center = rng.integers(0, m, size=(n_rows, 1))
        idx = (center + rng.integers(0, w, size=(n_rows, k))) % m
    else:
        raise ValueError(pattern)
    idx.sort(axis=1)
    for _ in range(1000):
        dup = np.any(idx[:, 1:] == idx[:, :-1], axis=1) if k > 1 else np.zeros(n_rows, bool)
        nd = int(dup.sum())
        if nd == 0:
            break
        if pattern == "uniform":
            new = rng.integers(0, m, size=(nd, k))
        else:
            w = min(window, m)
            c = rng.integers(0, m, size=(nd, 1))
            new = (c + rng.integers(0, w, size=(nd, k))) % m
        new.sort(axis=1)
        idx[dup] = new
    else:  # pragma: no cover
        raise RuntimeError("could not draw distinct indices")
    return idx


def g1_quasidefinite(n_s, n_d, m_E, m_I, seed, pattern="uniform", nnz_per_row=5,
                     private=True, scaled=True, delta_w=0.0, delta_c=0.0):
    """G1: quasi-definite MDS instance.

    Every constraint c gets one private sparse variable (single entry 1.0) so
    J_s^T W J_s >= diag(w_priv) > 0; the remaining n_s - m sparse variables each
    touch `nnz_per_row` distinct constraints (uniform, or bus-local window 64).
    H_dd = G G^T / n_d + I, so M_xx >= I and M_yy < 0: M is quasi-definite and
    inertia(M) = (n_d, 0, m) by closed form (Haynsworth).
    """
    rng = np.random.default_rng(seed)
    m = m_E + m_I
    n_priv = m if (private and m > 0) else 0
    if n_s < n_priv:
        n_priv = 0
    n_r = n_s - n_priv
    rho = max(nnz_per_row * max(n_s, 1) / max(m, 1), 1.0)
    k = min(nnz_per_row, m)
    idx = _distinct_rows(rng, n_r, k, m, pattern)
    vals = rng.standard_normal((n_r, k)) * (np.sqrt(1.0 / rho) if scaled else 1.0)
    # assemble rows: random rows, then private rows, then shuffle row order
    counts = np.concatenate([np.full(n_r, k, dtype=np.int64), np.ones(n_priv, dtype=np.int64)])
    cols = [idx.reshape(-1), np.arange(n_priv, dtype=np.int64)]
    vv = [vals.reshape(-1), np.ones(n_priv)]
    cols = np.concatenate(cols)
    vv = np.concatenate(vv)
    perm = rng.permutation(n_s)
    starts = np.concatenate([[0], np.cumsum(counts)])
    new_counts = counts[perm]
    rowptr = np.concatenate([[0], np.cumsum(new_counts)]).astype(np.int64)
    gather = _gather_runs(starts, perm, counts)
    colidx = cols[gather].astype(np.int32)
    val = vv[gather].astype(np.float64)
    h_ss = rng.uniform(0.0, 1.0, n_s)
    sigma_s = rng.uniform(0.5, 2.0, n_s)
    if n_d > 0:
        G = rng.standard_normal((n_d, n_d))
        H = np.asfortranarray(G @ G.T / n_d + np.eye(n_d))
    else:
        H = np.zeros((0, 0), order="F")
    sigma_d = rng.uniform(0.1, 1.0, n_d)
    J_d = np.asfortranarray(rng.standard_normal((m, n_d)) / np.sqrt(max(n_d, 1)))
    d_h = rng.uniform(1.0, 10.0, m_I)
    r = rng.standard_normal(n_s + n_d + m)
    return MDSProblem(n_s, n_d, m_E, m_I, rowptr.astype(np.int32), colidx, val, h_ss, sigma_s, H, sigma_d,
                      J_d, d_h, float(delta_w), float(delta_c), r, expected_inertia=(n_d, 0, m),
                      meta=dict(gen="G1", seed=seed, pattern=pattern, private=private, scaled=scaled))


def _gather_runs(starts, perm, counts):
    """Vectorised np.concatenate([arange(starts[p], starts[p]+counts[p]) for p in perm])."""
    c = counts[perm]
    tot = int(c.sum())
    if tot == 0:
        return np.zeros(0, dtype=np.int64)
    base = np.repeat(starts[perm] - np.concatenate([[0], np.cumsum(c)[:-1]]), c)
    return base + np.arange(tot)


def g2_indefinite(n_s, n_d, m_E, m_I, seed, p_neg, pattern="uniform", delta_c=1.0):
    """G2: indefinite MDS instance with closed-form inertia (n_d - p, 0, m + p).

    H_dd = U diag(lambda) U^T with p negative eigenvalues, |lambda| in [1,10];
    sigma_d = delta_w = 0; delta_c = 1 and ||J_d||_F^2 = delta_c/2, so the Schur
    complement -C - J_d A^{-1} J_d^T is negative definite (Haynsworth).
    """
    prob = g1_quasidefinite(n_s, n_d, m_E, m_I, seed, pattern=pattern)
    rng = np.random.default_rng(seed + 7919)
    Q, _ = np.linalg.qr(rng.standard_normal((n_d, n_d)))
    lam = rng.uniform(1.0, 10.0, n_d)
    lam[:p_neg] *= -1.0
    prob.H_dd = np.asfortranarray((Q * lam) @ Q.T)
    prob.sigma_d = np.zeros(n_d)
    prob.delta_w = 0.0
    prob.delta_c = float(delta_c)
    Jd = rng.standard_normal((n_d + m_E + m_I - n_d, n_d))
    Jd *= np.sqrt(delta_c / 2.0) / np.linalg.norm(Jd)
    prob.J_d = np.asfortranarray(Jd)
    prob.expected_inertia = (n_d - p_neg, 0, m_E + m_I + p_neg)
    prob.meta.update(gen="G2", p_neg=p_neg)
    return prob


def g6_negative_curvature(n_s, n_d, m_E, m_I, seed, lam_neg=(-1.0,), jd_norm=1e-3, pattern="uniform"):
    """G6 (inertia-correction workload): a G1 instance whose dense Hessian has
    prescribed negative eigenvalues.  H_dd = Q diag(lambda) Q^T with lambda_i =
    lam_neg[i] for the first len(lam_neg), U[1,10] otherwise; sigma_d = delta_w =
    delta_c = 0; J_d scaled to ||J_d||_F = jd_norm (weak coupling).  The G1
    y-block keeps C = J_s^T W J_s + D_h ~ O(1) positive definite, so by
    Haynsworth the inertia of M at a regularisation delta_w is, up to an
    O(jd_norm^2) shift of the crossover, (#{lambda+delta_w>0}, #{=0}, m+#{<0}):
    the smallest acceptable delta_w is -min(lambda) (meta["lam"])."""
    prob = g1_quasidefinite(n_s, n_d, m_E, m_I, seed, pattern=pattern)
    rng = np.random.default_rng(seed + 104729)
    Q, _ = np.linalg.qr(rng.standard_normal((n_d, n_d)))
    lam = rng.uniform(1.0, 10.0, n_d)
    lam[:len(lam_neg)] = np.asarray(lam_neg, dtype=np.float64)
    prob.H_dd = np.asfortranarray((Q * lam) @ Q.T)
    prob.sigma_d = np.zeros(n_d)
    prob.delta_w = 0.0
    prob.delta_c = 0.0
    Jd = rng.standard_normal((m_E + m_I, n_d))
    Jd *= jd_norm / np.linalg.norm(Jd)
    prob.J_d = np.asfortranarray(Jd)
    p = int(np.sum(lam < 0))
    prob.expected_inertia = (n_d - p, 0, m_E + m_I + p)
    prob.meta.update(gen="G6", lam=lam.copy())
    return prob


def g5_singular(n_s, n_d, m_E, m_I, seed):
    """G5: exactly singular M: equality row c0 has no J_s entries (its private
    variable removed) and a zero J_d row, delta_c = 0 -> M has an exactly zero
    row/column; expected inertia (n_d, 1, m-1)."""
    prob = g1_quasidefinite(n_s, n_d, m_E, m_I, seed)
    assert m_E >= 1
    c0 = 0
    keep = prob.colidx != c0
    counts = np.diff(prob.rowptr.astype(np.int64))
    row_of = np.repeat(np.arange(prob.n_s), counts)
    new_counts = np.bincount(row_of[keep], minlength=prob.n_s)
    prob.colidx = prob.colidx[keep].astype(np.int32)
    prob.val = prob.val[keep]
    prob.rowptr = np.concatenate([[0], np.cumsum(new_counts)]).astype(np.int32)
    Jd = np.array(prob.J_d)
    Jd[c0, :] = 0.0
    prob.J_d = np.asfortranarray(Jd)
    prob.delta_c = 0.0
    m = m_E + m_I
    prob.expected_inertia = (n_d, 1, m - 1)
    prob.meta.update(gen="G5", zero_row=n_d + c0)
    return prob


def g3_prescribed(N, seed, n2x2=None, n_reflectors=8):
    """G3: dense symmetric indefinite matrix with prescribed inertia (C5 stress).

    B = blockdiag of 1x1 +-10^U[0,3] and 2x2 [[e,1],[1,e']] (|e|<0.1, det<0),
    symmetrically permuted, then M = H_8..H_1 B H_1..H_8 (Householder
    reflectors).  Returns (M Fortran, (pos, zero, neg))."""
    rng = np.random.default_rng(seed)
    if n2x2 is None:
        n2x2 = N // 8
    n1 = N - 2 * n2x2
    B = np.zeros((N, N))
    sign = rng.choice([-1.0, 1.0], size=n1)
    lam = sign * 10.0 ** rng.uniform(0.0, 3.0, n1)
    pos = int((lam > 0).sum()) + n2x2
    neg = int((lam < 0).sum()) + n2x2
    i = 0
    for t in range(n1):
        B[i, i] = lam[t]
        i += 1
    for t in range(n2x2):
        e1, e2 = rng.uniform(-0.1, 0.1, 2)
        B[i, i], B[i + 1, i + 1] = e1, e2
        B[i, i + 1] = B[i + 1, i] = 1.0
        i += 2
    p = rng.permutation(N)
    B = B[np.ix_(p, p)]
    for _ in range(n_reflectors):
        v = rng.standard_normal(N)
        v /= np.linalg.norm(v)
        Bv = B @ v
        vBv = v @ Bv
        B = B - 2.0 * np.outer(v, Bv) - 2.0 * np.outer(Bv, v) + 4.0 * vBv * np.outer(v, v)
    B = 0.5 * (B + B.T)
    return np.asfortranarray(B), (pos, 0, neg)


def g3_prescribed_torch(N, seed, n2x2=None, n_reflectors=8, device="cuda"):
    """G3 built with torch on `device` (the C5 size, 8.6 GB, is impractical in
    numpy): the same random draws in the same order as g3_prescribed, the same
    reflectors, the same final symmetrisation.  Returns (M as a torch (N, N)
    float64 tensor, (pos, zero, neg))."""
    import torch
    rng = np.random.default_rng(seed)
    if n2x2 is None:
        n2x2 = N // 8
    n1 = N - 2 * n2x2
    sign = rng.choice([-1.0, 1.0], size=n1)
    lam = sign * 10.0 ** rng.uniform(0.0, 3.0, n1)
    pos = int((lam > 0).sum()) + n2x2
    neg = int((lam < 0).sum()) + n2x2
    diag = np.zeros(N)
    off = np.zeros(N)            # off[i] = B[i, i+1] = B[i+1, i]
    diag[:n1] = lam
    i = n1
    for t in range(n2x2):
        e1, e2 = rng.uniform(-0.1, 0.1, 2)
        diag[i], diag[i + 1] = e1, e2
        off[i] = 1.0
        i += 2
    p = rng.permutation(N)
    f64 = dict(dtype=torch.float64, device=device)
    B = torch.zeros((N, N), **f64)
    idx = torch.arange(N, device=device)
    B[idx, idx] = torch.as_tensor(diag, **f64)
    j = torch.as_tensor(np.nonzero(off)[0], device=device)
    B[j, j + 1] = 1.0
    B[j + 1, j] = 1.0
    pt = torch.as_tensor(p, device=device)
    B = B[pt][:, pt]
    for _ in range(n_reflectors):
        v = rng.standard_normal(N)
        v /= np.linalg.norm(v)
        vt = torch.as_tensor(v, **f64)
        Bv = B @ vt
        vBv = float(vt @ Bv)
        B.addr_(vt, Bv, alpha=-2.0)
        B.addr_(Bv, vt, alpha=-2.0)
        B.addr_(vt, vt, alpha=4.0 * vBv)
    B = 0.5 * (B + B.T)
    return B, (pos, 0, neg)


def g4_random_symmetric(N, seed, shrink_diag=False):
    """G4: B + B^T (inertia by eigvalsh in tests); optional shrunken diagonal to force 2x2 pivots."""
    rng = np.random.default_rng(seed)
    B = rng.standard_normal((N, N))
    A = B + B.T
    if shrink_diag:
        A[np.diag_indices(N)] *= 0.01
    return np.asfortranarray(A)


@dataclass
class StepVectors:
    """Inputs of the barrier vector kernels (K1): primal x (incl. slacks) and its
    bound duals, search direction, bounds with +-1e20 sentinels."""
    x: np.ndarray
    dx: np.ndarray
    lo: np.ndarray
    up: np.ndarray
    zl: np.ndarray
    zu: np.ndarray
    dzl: np.ndarray
    dzu: np.ndarray
    tau: float
    mu: float


def step_vectors(n, seed, frac_lo=0.5, frac_up=0.5, mu=0.1):
    """Strictly interior iterate with a mix of finite / infinite bounds.
    Duals of infinite bounds are 0 (they never enter any formula)."""
    rng = np.random.default_rng(seed)
    has_lo = rng.random(n) < frac_lo
    has_up = rng.random(n) < frac_up
    x = rng.uniform(-5.0, 5.0, n)
    lo = np.where(has_lo, x - rng.uniform(0.01, 3.0, n), -INF)
    up = np.where(has_up, x + rng.uniform(0.01, 3.0, n), INF)
    zl = np.where(has_lo, rng.uniform(0.01, 2.0, n), 0.0)
    zu = np.where(has_up, rng.uniform(0.01, 2.0, n), 0.0)
    dx = rng.standard_normal(n) * 2.0
    dzl = rng.standard_normal(n)
    dzu = rng.standard_normal(n)
    tau = max(0.99, 1.0 - mu)
    return StepVectors(x, dx, lo, up, zl, zu, dzl, dzu, tau, mu)


def config_problem(cfg: str, seed: Optional[int] = None, pattern="uniform", instance=0):
    """Concrete G1 instance of BASELINE.json config C1..C4 (seed = 1000*cfg + instance)."""
    shp = CONFIGS[cfg]
    if seed is None:
        seed = 1000 * int(cfg[1:]) + instance
    return g1_quasidefinite(shp["n_s"], shp["n_d"], shp["m_E"], shp["m_I"], seed, pattern=pattern)


def step_vectors_for(prob: MDSProblem, seed: int, mu=0.1):
    """K1 inputs for the primal block (x_s, x_d): n_b = n_s + n_d components
    (the primal direction itself comes from the solve)."""
    return step_vectors(prob.n_s + prob.n_d, seed, mu=mu)


def scopf_base(seed=4000, n_s=131_072, n_d=1024, m_E=512, m_I=512, pattern="local"):
    """C4 base case: one G1 instance whose sparsity pattern all contingency
    scenarios share (SCOPF: the same network with one element altered)."""
    return g1_quasidefinite(n_s, n_d, m_E, m_I, seed, pattern=pattern)


def scopf_scenario(base: MDSProblem, s: int, seed: int = 4000):
    """Contingency scenario s of a SCOPF batch: same pattern
    as `base`, values re-drawn with seed (seed, s) so that the G1 structure --
    hence the closed-form inertia (n_d, 0, m) -- is preserved:
      J_s values scaled by U[0.8,1.2] (private entries kept at 1.0), h_ss, sigma_s,
      sigma_d, d_h, r re-drawn, H_dd + diag(U[0,0.1]), J_d scaled by U[0.9,1.1]."""
    rng = np.random.default_rng([seed, s])
    n_s, n_d, m = base.n_s, base.n_d, base.m
    scale = rng.uniform(0.8, 1.2, base.nnz)
    val = np.where(base.val == 1.0, 1.0, base.val * scale)
    H = np.array(base.H_dd, order="F", copy=True)
    H[np.diag_indices(n_d)] += rng.uniform(0.0, 0.1, n_d)
    J_d = np.asfortranarray(np.asarray(base.J_d) * rng.uniform(0.9, 1.1, (m, n_d)))
    return MDSProblem(n_s, n_d, base.m_E, base.m_I, base.rowptr, base.colidx, val,
                      rng.uniform(0.0, 1.0, n_s), rng.uniform(0.5, 2.0, n_s), H, rng.uniform(0.1, 1.0, n_d),
                      J_d, rng.uniform(1.0, 10.0, base.m_I), 0.0, 0.0, rng.standard_normal(n_s + n_d + m),
                      expected_inertia=(n_d, 0, m), meta=dict(gen="SCOPF", seed=seed, scenario=s))


# ----------------------------------------------------------------------------- convex QP (C3 IPM workload)
@dataclass
class QPProblem:
    """Convex QP in MDS form (SURVEY.md §8(d) "C3 full IPM workload"):
        min  1/2 x_d^T H_dd x_d + 1/2 sum h_ss x_s^2 + c^T x
        s.t. J_E x = g_E,   h_l <= J_I x <= h_u,   lo <= x <= up
    with J = [J_s^T  J_d] (J_s CSR n_s x m, rows = sparse variables, reading R1),
    built around a strictly interior x_star.  Infinite bounds are +-1e20 (R10).
    `base` carries the pattern and the Hessian / Jacobian values (an MDSProblem
    whose sigma_s, sigma_d, d_h, r are unused placeholders)."""
    base: MDSProblem
    c: np.ndarray          # f64[n]
    g_E: np.ndarray        # f64[m_E]
    h_l: np.ndarray        # f64[m_I]
    h_u: np.ndarray        # f64[m_I]
    lo: np.ndarray         # f64[n]
    up: np.ndarray         # f64[n]
    x_star: np.ndarray     # f64[n] strictly interior, feasible

    @property
    def n(self):
        return self.base.n_s + self.base.n_d


def _jac_times(prob: MDSProblem, x):
    """(J x)_c = sum_k J_s[k, c] x_s[k] + (J_d x_d)_c  -- input construction only."""
    n_s = prob.n_s
    rows = np.repeat(np.arange(n_s), np.diff(prob.rowptr))
    out = np.bincount(prob.colidx, weights=prob.val * x[:n_s][rows], minlength=prob.m)
    if prob.n_d and prob.m:
        out = out + np.asarray(prob.J_d) @ x[n_s:]
    return out


def qp_problem(n_s, n_d, m_E, m_I, seed, pattern="uniform", box_frac=0.5, c_scale=1.0):
    """Seeded convex QP with the G1 structure (private sparse variable per constraint,
    H_dd = G G^T/n_d + I, h_ss ~ U[0.1, 1] so every sparse variable has curvature)."""
    base = g1_quasidefinite(n_s, n_d, m_E, m_I, seed, pattern=pattern)
    rng = np.random.default_rng([seed, 77])
    n = n_s + n_d
    base.h_ss = rng.uniform(0.1, 1.0, n_s)
    x_star = rng.uniform(-5.0, 5.0, n)
    boxed = rng.random(n) < box_frac
    lo = np.where(boxed, -10.0, -INF)
    up = np.where(boxed, 10.0, INF)
    c = rng.standard_normal(n) * c_scale
    Jx = _jac_times(base, x_star)
    g_E = Jx[:m_E].copy()
    h_l = Jx[m_E:] - rng.uniform(0.5, 2.0, m_I)
    h_u = Jx[m_E:] + rng.uniform(0.5, 2.0, m_I)
    base.meta = dict(base.meta, gen="QP", seed=seed)
    return QPProblem(base, c, g_E, h_l, h_u, lo, up, x_star)


def qp_config(cfg: str, seed: Optional[int] = None, pattern="uniform"):
    """The QP of BASELINE.json config C1..C3 shapes (seed = 1000*cfg + 500)."""
    shp = CONFIGS[cfg]
    if seed is None:
        seed = 1000 * int(cfg[1:]) + 500
    return qp_problem(shp["n_s"], shp["n_d"], shp["m_E"], shp["m_I"], seed, pattern=pattern)


def synthetic_problem(k: int):
    """The paper's mini-app problem nlpMDS_ex4 ("a convex optimization
    problem with m = n_s + 3 constraints ... n_d = n_s = k ... compressed matrix of
    size (2k+3) x (2k+3)"), with the model of SPEC.md:288-297:
      f = 1/2 sum (x_s,i - 1)^2 + 1/2 x_d^T (I + e e^T / k) x_d - e^T x_d
      (1/k) sum x_s + (1/k) sum x_d = 1,   x_s,1 - x_d,1 = 0                  (m_E = 2)
      x_s,i + (1/k) sum_j x_d,j <= 2  (i = 1..k),  0.5 <= (1/k) sum_j x_d,j <= 3  (m_I = k + 1)
      -10 <= x_s, x_d <= 10
    as a QPProblem in MDS form (J_s rows = sparse variables, reading R1; the constant
    k/2 of f dropped).  x_star is the interior start x_s = 0.5, x_d = 1 (slacks
    strictly inside their bounds; the equalities are not satisfied there)."""
    if k < 1:
        raise ValueError("k >= 1")
    n_s = n_d = k
    m_E, m_I = 2, k + 1
    m = m_E + m_I
    rows, cols, vals = [], [], []
    for i in range(k):
        ent = [(0, 1.0 / k)]
        if i == 0:
            ent.append((1, 1.0))
        ent.append((2 + i, 1.0))
        for c, v in ent:
            rows.append(i)
            cols.append(c)
            vals.append(v)
    rowptr = np.zeros(n_s + 1, dtype=np.int64)
    np.add.at(rowptr, np.asarray(rows) + 1, 1)
    rowptr = np.cumsum(rowptr).astype(np.int32)
    colidx = np.asarray(cols, dtype=np.int32)
    val = np.asarray(vals, dtype=np.float64)
    H = np.asfortranarray(np.eye(n_d) + np.full((n_d, n_d), 1.0 / k))
    J_d = np.zeros((m, n_d), order="F")
    J_d[0, :] = 1.0 / k
    J_d[1, 0] = -1.0
    J_d[2:, :] = 1.0 / k
    base = MDSProblem(n_s, n_d, m_E, m_I, rowptr, colidx, val, np.ones(n_s), np.zeros(n_s), H, np.zeros(n_d),
                      J_d, np.ones(m_I), 0.0, 0.0, np.zeros(n_s + n_d + m),
                      meta=dict(gen="nlpMDS_ex4", k=k))
    c = np.concatenate([-np.ones(n_s), -np.ones(n_d)])
    g_E = np.array([1.0, 0.0])
    h_l = np.concatenate([np.full(k, -INF), [0.5]])
    h_u = np.concatenate([np.full(k, 2.0), [3.0]])
    lo = np.full(n_s + n_d, -10.0)
    up = np.full(n_s + n_d, 10.0)
    start = np.concatenate([np.full(n_s, 0.5), np.full(n_d, 1.0)])
    return QPProblem(base, c, g_E, h_l, h_u, lo, up, start)
