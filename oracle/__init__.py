"""CPU oracle for the condensed-KKT hot path — TEST INFRASTRUCTURE ONLY.

Plain C (``oracle.c``, gcc ``-O2 -ffp-contract=off``) behind ctypes, following
PAPER.md §2 (Eq.(5)-(6)) step by step.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product package
``paper_2605_13736_b200`` never imports it and shares no code with it.

Every function here is pinned by ``tests/test_oracle_*.py`` (``-m "not gpu"``)
against values the paper / SPEC examples fix, closed forms, LAPACK (scipy) and
brute force; see DESIGN.md §Oracle pins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK, ERR_ARG, ERR_PATTERN, ERR_NONPOSITIVE, ERR_NONFINITE, ERR_SINGULAR, ERR_NOT_INTERIOR = 0, -1, -2, -3, -4, -5, -6
ALPHA_BK = (1.0 + np.sqrt(17.0)) / 8.0


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (plain gcc, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-std=c99", "-shared", "-fPIC",
               "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P, I64, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double
            L.or_condense.restype = ctypes.c_int
            L.or_condense.argtypes = [I64, I64, I64, I64, P, P, P, P, P, P, I64, P, P, I64, P, D, D, P, P, I64, P, P]
            L.or_anorm_lower.restype = ctypes.c_int
            L.or_anorm_lower.argtypes = [I64, P, I64, P]
            L.or_ldlt_nopiv.restype = ctypes.c_int
            L.or_ldlt_nopiv.argtypes = [I64, P, I64, D]
            L.or_bk_factor.restype = I64
            L.or_bk_factor.argtypes = [I64, P, I64, P]
            L.or_inertia.restype = ctypes.c_int
            L.or_inertia.argtypes = [I64, P, I64, P, D, P]
            L.or_bk_solve.restype = ctypes.c_int
            L.or_bk_solve.argtypes = [I64, P, I64, P, P, D]
            L.or_recover.restype = None
            L.or_recover.argtypes = [I64, P, P, P, P, P, P, P]
            L.or_step_vectors.restype = ctypes.c_int
            L.or_step_vectors.argtypes = [I64, P, P, P, P, P, P, P, P, D, D, P, P]
            L.or_num_threads.restype = ctypes.c_int
            L.or_set_threads.argtypes = [ctypes.c_int]
            L.or_set_threads.restype = None
            L.or_norm_inf.restype = D
            L.or_norm_inf.argtypes = [I64, P]
            _lib = L
    return _lib


def num_threads() -> int:
    """Threads the BK factorization's column loop uses (OpenMP; bit-identical for any count)."""
    return int(lib().or_num_threads())


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _fortran(a):
    return np.asfortranarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, code, what=""):
        super().__init__(f"oracle status {code} {what}")
        self.code = code


def condense(prob, with_rhs: bool = True):
    """O1 (Eq.(5)->Eq.(6)).  Returns (M lower, col-major N x N, rhs_c, w)."""
    n_s, n_d, m_E, m_I = prob.n_s, prob.n_d, prob.m_E, prob.m_I
    N = n_d + m_E + m_I
    M = np.zeros((N, N), dtype=np.float64, order="F")
    rhs = np.zeros(N) if with_rhs else None
    w = np.zeros(max(n_s, 1))
    rowptr = np.ascontiguousarray(prob.rowptr, dtype=np.int32)
    colidx = np.ascontiguousarray(prob.colidx, dtype=np.int32)
    val = _f64(prob.val)
    H = _fortran(prob.H_dd) if n_d > 0 else np.zeros((1, 1), order="F")
    Jd = _fortran(prob.J_d) if n_d > 0 and N - n_d > 0 else np.zeros((1, 1), order="F")
    dh = _f64(prob.d_h) if m_I > 0 else np.ones(1)
    r = _f64(prob.r) if with_rhs else None
    st = lib().or_condense(n_s, n_d, m_E, m_I, _p(rowptr), _p(colidx), _p(val), _p(_f64(prob.h_ss)),
                           _p(_f64(prob.sigma_s)), _p(H), max(H.shape[0], 1), _p(_f64(prob.sigma_d)),
                           _p(Jd), max(Jd.shape[0], 1), _p(dh), float(prob.delta_w), float(prob.delta_c),
                           _p(r), _p(M), max(N, 1), _p(rhs), _p(w))
    if st != OK:
        raise OracleError(st, "condense")
    return M, rhs, w[:n_s]


def anorm_lower(A):
    A = _fortran(A)
    out = np.zeros(1)
    st = lib().or_anorm_lower(A.shape[0], _p(A), max(A.shape[0], 1), _p(out))
    if st != OK:
        raise OracleError(st, "anorm")
    return float(out[0])


def default_tol(A):
    """Zero-pivot tolerance tol = N * eps * ||A||_inf (reading R4)."""
    return A.shape[0] * np.finfo(np.float64).eps * anorm_lower(A)


def ldlt_nopiv(A, tol=None):
    """O2: unpivoted LDL^T in place on a copy.  Returns LD (col-major)."""
    A = np.array(A, dtype=np.float64, order="F", copy=True)
    tol = default_tol(A) if tol is None else tol
    st = lib().or_ldlt_nopiv(A.shape[0], _p(A), max(A.shape[0], 1), tol)
    if st != OK:
        raise OracleError(st, "ldlt_nopiv")
    return A


def bk_factor(A):
    """O3: Bunch-Kaufman (dsytf2 'L').  Returns (LD, ipiv 1-based LAPACK encoding, info)."""
    A = np.array(A, dtype=np.float64, order="F", copy=True)
    N = A.shape[0]
    ipiv = np.zeros(max(N, 1), dtype=np.int32)
    info = lib().or_bk_factor(N, _p(A), max(N, 1), _p(ipiv))
    return A, ipiv[:N], int(info)


def inertia(LD, ipiv, tol):
    out = np.zeros(3, dtype=np.int64)
    st = lib().or_inertia(LD.shape[0], _p(_fortran(LD)), max(LD.shape[0], 1), _p(np.ascontiguousarray(ipiv, dtype=np.int32)), float(tol), _p(out))
    if st != OK:
        raise OracleError(st, "inertia")
    return tuple(int(v) for v in out)


def bk_solve(LD, ipiv, b, tol):
    LD = _fortran(LD)
    x = np.array(b, dtype=np.float64, copy=True)
    st = lib().or_bk_solve(LD.shape[0], _p(LD), max(LD.shape[0], 1), _p(np.ascontiguousarray(ipiv, dtype=np.int32)), _p(x), float(tol))
    if st != OK:
        raise OracleError(st, "bk_solve")
    return x


def recover(prob, w, r_xs, dy):
    dx = np.zeros(max(prob.n_s, 1))
    lib().or_recover(prob.n_s, _p(np.ascontiguousarray(prob.rowptr, dtype=np.int32)),
                     _p(np.ascontiguousarray(prob.colidx, dtype=np.int32)), _p(_f64(prob.val)),
                     _p(_f64(w)), _p(_f64(r_xs)), _p(_f64(dy)), _p(dx))
    return dx[:prob.n_s]


def step_vectors(x, dx, lo, up, zl, zu, dzl, dzu, tau, mu, want_sigma=True):
    """O7.  Returns (status, dict(alpha_p, alpha_d, compl_inf, compl_sum, n_compl, first_bad), sigma)."""
    n = len(x)
    out = np.zeros(6)
    sig = np.zeros(max(n, 1)) if want_sigma else None
    arrs = [_f64(v) for v in (x, dx, lo, up, zl, zu, dzl, dzu)]
    st = lib().or_step_vectors(n, *[_p(a) for a in arrs], float(tau), float(mu), _p(out), _p(sig))
    res = dict(alpha_p=out[0], alpha_d=out[1], compl_inf=out[2], compl_sum=out[3],
               n_compl=int(out[4]), first_bad=int(out[5]))
    return st, res, (sig[:n] if want_sigma else None)


def norm_inf(v):
    v = _f64(v)
    return float(lib().or_norm_inf(len(v), _p(v)))


def newton_step(prob, tol=None):
    """The whole hot path on the CPU, in the paper's order (Fig.1 PAPER.md:53-58,
    §2.2-2.3): condense -> BK factor -> inertia -> solve -> recover dx_s.
    Returns dict with M, rhs_c, w, LD, ipiv, inertia, dxy (=dx_d,dy), dx_s."""
    M, rhs, w = condense(prob)
    N = M.shape[0]
    tol = default_tol(M) if tol is None else tol
    LD, ipiv, info = bk_factor(M)
    ine = inertia(LD, ipiv, tol)
    dxy = bk_solve(LD, ipiv, rhs, tol)
    dx_s = recover(prob, w, np.asarray(prob.r)[:prob.n_s], dxy[prob.n_d:])
    return dict(M=M, rhs_c=rhs, w=w, LD=LD, ipiv=ipiv, info=info, inertia=ine, dxy=dxy, dx_s=dx_s, tol=tol)


# ----------------------------------------------------------------------------- inertia correction
IC_DEFAULTS = dict(delta_w0=1e-4, delta_w_min=1e-20, delta_w_max=1e40, kappa_w_plus=8.0, kappa_w_plus_first=100.0,
                   kappa_w_minus=1.0 / 3.0, delta_c_bar=1e-8, kappa_c=0.25)


def factor_inertia(prob, tol=None):
    """O1 + O3 + O4 for one regularisation (prob.delta_w, prob.delta_c): (inertia, M, LD, ipiv, tol)."""
    M, rhs, w = condense(prob)
    tol = default_tol(M) if tol is None else tol
    LD, ipiv, _ = bk_factor(M)
    return inertia(LD, ipiv, tol), dict(M=M, rhs=rhs, w=w, LD=LD, ipiv=ipiv, tol=tol)


def inertia_correction(prob, mu, delta_w_last=0.0, params=None):
    """Inertia correction, written out step by step (PAPER.md:161 -- regularise
    with increasingly large multiples until the inertia of Eq.(5) is (n,0,m);
    by PAPER.md:191 the condensed target is (n_d,0,m)), with the multiples of the
    algorithm the paper cites for it (Wachter & Biegler 2006 Algorithm IC,
    constants SPEC.md:354; reading R22):
      IC-1 (0,0); IC-2 delta_c = delta_c_bar mu^kappa_c iff zero eigenvalues;
      IC-3 delta_w = delta_w0 (delta_w_last = 0) or max(delta_w_min, kappa_w_minus delta_w_last);
      IC-4 accept on target inertia; IC-5 delta_w *= kappa_w_plus_first (delta_w_last = 0) or
      kappa_w_plus; IC-6 delta_w > delta_w_max -> singular.
    Returns dict(delta_w, delta_c, delta_w_last, trials=[(dw, dc, inertia)], dxy, dx_s, inertia)."""
    import dataclasses
    P = dict(IC_DEFAULTS, **(params or {}))
    target = (prob.n_d, 0, prob.m_E + prob.m_I)
    trials = []

    def attempt(dw, dc):
        q = dataclasses.replace(prob, delta_w=float(dw), delta_c=float(dc))
        ine, f = factor_inertia(q)
        trials.append((float(dw), float(dc), ine))
        return q, ine, f

    q, ine, f = attempt(0.0, 0.0)
    dw = dc = 0.0
    if ine != target:
        dc = P["delta_c_bar"] * mu ** P["kappa_c"] if ine[1] > 0 else 0.0
        dw = P["delta_w0"] if delta_w_last == 0.0 else max(P["delta_w_min"], P["kappa_w_minus"] * delta_w_last)
        while True:
            q, ine, f = attempt(dw, dc)
            if ine == target:
                delta_w_last = dw
                break
            dw *= P["kappa_w_plus_first"] if delta_w_last == 0.0 else P["kappa_w_plus"]
            if dw > P["delta_w_max"]:
                raise OracleError(ERR_SINGULAR, "inertia correction: delta_w > delta_w_max")
    dxy = bk_solve(f["LD"], f["ipiv"], f["rhs"], f["tol"])
    dx_s = recover(q, f["w"], np.asarray(q.r)[:q.n_s], dxy[q.n_d:])
    return dict(delta_w=dw, delta_c=dc, delta_w_last=delta_w_last, trials=trials, inertia=ine, dxy=dxy, dx_s=dx_s)


# ----------------------------------------------------------------------------- K2 mat-vec
def kkt_matvec(prob, x):
    """K x for the full (uncondensed) Eq.(5) matrix, x laid out
    [x_s | x_d | y_g | y_h]: the block definition written out with library
    products (scipy CSR mat-vec for J_s, numpy for the dense blocks; H_dd from its
    lower triangle, R14):
      (Kx)_s = (h_ss + sigma_s + delta_w) x_s + J_s y
      (Kx)_d = (H_dd + diag(sigma_d) + delta_w I) x_d + J_d^T y
      (Kx)_y = J_s^T x_s + J_d x_d - (diag(0_{m_E}, 1/d_h) + delta_c I) y"""
    import scipy.sparse as sp
    n_s, n_d, m_E, m_I = prob.n_s, prob.n_d, prob.m_E, prob.m_I
    m = m_E + m_I
    x = np.asarray(x, dtype=np.float64)
    xs, xd, y = x[:n_s], x[n_s:n_s + n_d], x[n_s + n_d:]
    Js = sp.csr_matrix((np.asarray(prob.val, dtype=np.float64), np.asarray(prob.colidx), np.asarray(prob.rowptr)),
                       shape=(n_s, m))
    H = np.asarray(prob.H_dd, dtype=np.float64)
    Hs = np.tril(H) + np.tril(H, -1).T if n_d else np.zeros((0, 0))
    Jd = np.asarray(prob.J_d, dtype=np.float64).reshape(m, n_d) if n_d and m else np.zeros((m, n_d))
    ks = (np.asarray(prob.h_ss) + np.asarray(prob.sigma_s) + prob.delta_w) * xs + Js @ y
    kd = Hs @ xd + (np.asarray(prob.sigma_d) + prob.delta_w) * xd + Jd.T @ y
    dy = np.concatenate([np.zeros(m_E), 1.0 / np.asarray(prob.d_h, dtype=np.float64)]) + prob.delta_c
    ky = Js.T @ xs + Jd @ xd - dy * y
    return np.concatenate([ks, kd, ky])
