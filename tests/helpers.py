"""Test-only helpers: brute-force dense constructions used to PIN the oracle.

Nothing here is imported by the product package or by the oracle.
"""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def dense_js(prob):
    """Densify J_s (n_s x m) from CSR."""
    J = np.zeros((prob.n_s, prob.m))
    for k in range(prob.n_s):
        for p in range(prob.rowptr[k], prob.rowptr[k + 1]):
            J[k, prob.colidx[p]] += prob.val[p]
    return J


def full_kkt4(prob):
    """Assemble the full 4x4 block system of Eq.(5) densely,
    with delta_w on both Hessian blocks and -delta_c on both constraint blocks
    (PAPER.md:161).  Unknown order (x_s, x_d, y_g, y_h)."""
    n_s, n_d, m = prob.n_s, prob.n_d, prob.m
    n = n_s + n_d + m
    K = np.zeros((n, n))
    Js = dense_js(prob)
    q = prob.h_ss + prob.sigma_s + prob.delta_w
    K[:n_s, :n_s] = np.diag(q)
    H = np.array(prob.H_dd)
    Hs = np.tril(H) + np.tril(H, -1).T
    K[n_s:n_s + n_d, n_s:n_s + n_d] = Hs + np.diag(prob.sigma_d) + prob.delta_w * np.eye(n_d)
    K[n_s + n_d:, :n_s] = Js.T
    K[:n_s, n_s + n_d:] = Js
    K[n_s + n_d:, n_s:n_s + n_d] = prob.J_d
    K[n_s:n_s + n_d, n_s + n_d:] = np.asarray(prob.J_d).T
    yy = -prob.delta_c * np.ones(m)
    yy[prob.m_E:] -= 1.0 / prob.d_h
    K[n_s + n_d:, n_s + n_d:] = np.diag(yy)
    return K


def sym_from_lower(M):
    M = np.array(M)
    return np.tril(M) + np.tril(M, -1).T


def inertia_eig(A, tol=None):
    ev = np.linalg.eigvalsh(sym_from_lower(A))
    if tol is None:
        tol = A.shape[0] * np.finfo(float).eps * np.abs(ev).max() if A.size else 0.0
    return (int((ev > tol).sum()), int((np.abs(ev) <= tol).sum()), int((ev < -tol).sum()))


def bk_reconstruct(LD, ipiv):
    """Rebuild A from LAPACK-'L' product-form BK factors (dsytrf documentation:
    A = L D L^T, L = P(1) L(1) P(2) L(2) ..., each L(k) unit lower with the
    multipliers of the 1x1 / 2x2 pivot in columns k (k+1)).  Independent of
    the oracle's solve."""
    N = LD.shape[0]
    X = np.eye(N)
    D = np.zeros((N, N))
    k = 0
    while k < N:
        P = np.eye(N)
        if ipiv[k] > 0:
            kp = ipiv[k] - 1
            P[[k, kp]] = P[[kp, k]]
            Lk = np.eye(N)
            Lk[k + 1:, k] = LD[k + 1:, k]
            D[k, k] = LD[k, k]
            X = X @ P @ Lk
            k += 1
        else:
            kp = -ipiv[k] - 1
            P[[k + 1, kp]] = P[[kp, k + 1]]
            Lk = np.eye(N)
            Lk[k + 2:, k] = LD[k + 2:, k]
            Lk[k + 2:, k + 1] = LD[k + 2:, k + 1]
            D[k, k] = LD[k, k]
            D[k + 1, k] = D[k, k + 1] = LD[k + 1, k]
            D[k + 1, k + 1] = LD[k + 1, k + 1]
            X = X @ P @ Lk
            k += 2
    return X @ D @ X.T


def rel_inf(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = max(np.abs(b).max(), 1e-300) if b.size else 1.0
    return np.abs(a - b).max() / den if a.size else 0.0


def dense_qp_parts(qp):
    """(H, J) of a mdsgen.QPProblem assembled densely from its blocks (test-only)."""
    b = qp.base
    Js = dense_js(b)                                          # n_s x m
    n_s, n_d, m = b.n_s, b.n_d, b.m
    H = np.zeros((n_s + n_d, n_s + n_d))
    H[:n_s, :n_s] = np.diag(b.h_ss)
    if n_d:
        Hd = np.asarray(b.H_dd)
        H[n_s:, n_s:] = np.tril(Hd) + np.tril(Hd, -1).T
    J = np.zeros((m, n_s + n_d))
    J[:, :n_s] = Js.T
    if n_d and m:
        J[:, n_s:] = np.asarray(b.J_d)
    return H, J
