"""Pins for oracle O2 (unpivoted LDL^T), O3 (Bunch-Kaufman, dsytf2 'L'),
O4 (inertia) and O5 (solve, dsytrs 'L').  Pinned against LAPACK via scipy
(same algorithm: pivots must agree exactly), eigenvalue sign counts,
closed-form-inertia generators, an independent product-form reconstruction,
and the SPEC examples."""
import numpy as np
import pytest
import scipy.linalg
from scipy.linalg import lapack

import mdsgen
import oracle
from tests.helpers import bk_reconstruct, inertia_eig, rel_inf, sym_from_lower


def _lapack_bk(A):
    ldu, ipiv, info = lapack.dsytrf(np.array(A, order="F"), lower=1)
    return ldu, ipiv, info


@pytest.mark.parametrize("seed", range(60))
def test_bk_matches_lapack_dsytrf_pivots(seed):
    n = 3 + seed % 37
    A = mdsgen.g4_random_symmetric(n, seed, shrink_diag=(seed % 3 == 0))
    LD, ipiv, info = oracle.bk_factor(A)
    ldu, ipiv_l, info_l = _lapack_bk(A)
    assert info == info_l == 0
    np.testing.assert_array_equal(ipiv, ipiv_l)
    # L and D agree with LAPACK (product form) to rounding
    assert rel_inf(np.tril(LD), np.tril(ldu)) <= 1e-10


@pytest.mark.parametrize("n", [100, 200, 300])
def test_bk_matches_blocked_lapack_larger(n):
    A = mdsgen.g4_random_symmetric(n, 7 * n, shrink_diag=True)
    LD, ipiv, _ = oracle.bk_factor(A)
    _, ipiv_l, _ = _lapack_bk(A)
    np.testing.assert_array_equal(ipiv, ipiv_l)


def test_bk_spec_examples():
    # SPEC.md:208-210
    LD, ipiv, info = oracle.bk_factor(np.eye(3))
    np.testing.assert_array_equal(ipiv, [1, 2, 3]); assert info == 0
    assert oracle.inertia(LD, ipiv, 0.0) == (3, 0, 0)
    LD, ipiv, _ = oracle.bk_factor(np.diag([-1.0, -2.0]))
    assert oracle.inertia(LD, ipiv, 0.0) == (0, 0, 2)
    LD, ipiv, _ = oracle.bk_factor(np.array([[0.0, 1.0], [1.0, 0.0]]))
    np.testing.assert_array_equal(ipiv, [-2, -2])     # one 2x2 pivot (LAPACK gives the same)
    assert LD[0, 0] * LD[1, 1] - LD[1, 0] ** 2 == -1.0   # det -1
    assert oracle.inertia(LD, ipiv, 0.0) == (1, 0, 1)
    # SPEC.md:226-227
    LD, ipiv, _ = oracle.bk_factor(np.eye(4))
    assert oracle.inertia(LD, ipiv, 0.0) == (4, 0, 0)


@pytest.mark.parametrize("seed", range(25))
def test_bk_reconstruction_and_inertia_vs_eig(seed):
    # ||P L D L^T P^T - A|| <= 100 N eps ||A||; inertia == eigvalsh sign count
    n = 5 + 8 * seed
    A = mdsgen.g4_random_symmetric(n, 500 + seed, shrink_diag=(seed % 2 == 0))
    LD, ipiv, _ = oracle.bk_factor(A)
    R = bk_reconstruct(LD, ipiv)
    As = sym_from_lower(A)
    assert np.abs(R - As).max() <= 100 * n * np.finfo(float).eps * np.abs(As).sum(1).max()
    tol = oracle.default_tol(A)
    assert oracle.inertia(LD, ipiv, tol) == inertia_eig(A)


def test_sylvester_invariance():
    # inertia(S^T A S) == inertia(A) for nonsingular S
    rng = np.random.default_rng(11)
    for t in range(10):
        n = 30 + t
        A = mdsgen.g4_random_symmetric(n, 900 + t)
        S = rng.standard_normal((n, n)) + 3 * np.eye(n)
        B = S.T @ sym_from_lower(A) @ S
        B = 0.5 * (B + B.T)
        ia = oracle.inertia(*oracle.bk_factor(A)[:2], oracle.default_tol(A))
        ib = oracle.inertia(*oracle.bk_factor(B)[:2], oracle.default_tol(B))
        assert ia == ib


@pytest.mark.parametrize("N,n2", [(64, 8), (200, 40), (400, 100)])
def test_prescribed_spectrum_closed_form(N, n2):
    # G3: inertia fixed by construction; 2x2 branch exercised
    A, ine = mdsgen.g3_prescribed(N, seed=N, n2x2=n2)
    LD, ipiv, info = oracle.bk_factor(A)
    assert info == 0
    assert oracle.inertia(LD, ipiv, oracle.default_tol(A)) == ine
    assert (ipiv < 0).sum() > 0


@pytest.mark.parametrize("shape", [(400, 20, 10, 10), (3000, 96, 40, 40)])
def test_quasidefinite_closed_form_and_nopiv_agrees(shape):
    prob = mdsgen.g1_quasidefinite(*shape, seed=77)
    M, rhs, _ = oracle.condense(prob)
    tol = oracle.default_tol(M)
    LD, ipiv, info = oracle.bk_factor(M)
    assert oracle.inertia(LD, ipiv, tol) == prob.expected_inertia == (prob.n_d, 0, prob.m)
    # O2 unpivoted reference: same inertia (signs of D) and same solution
    LDn = oracle.ldlt_nopiv(M)
    d = np.diag(LDn)
    assert ((d > tol).sum(), 0, (d < -tol).sum()) == prob.expected_inertia
    x_bk = oracle.bk_solve(LD, ipiv, rhs, tol)
    # unpivoted solve by numpy triangular solves on the O2 factors (test-side)
    L = np.tril(LDn, -1) + np.eye(M.shape[0])
    y = scipy.linalg.solve_triangular(L, rhs, lower=True, unit_diagonal=True)
    x_np = scipy.linalg.solve_triangular(L.T, y / d, lower=False, unit_diagonal=True)
    assert rel_inf(x_bk, x_np) <= 1e-11


def test_indefinite_closed_form():
    prob = mdsgen.g2_indefinite(300, 60, 20, 20, seed=5, p_neg=7)
    M, _, _ = oracle.condense(prob)
    LD, ipiv, _ = oracle.bk_factor(M)
    assert oracle.inertia(LD, ipiv, oracle.default_tol(M)) == prob.expected_inertia == (53, 0, 47)
    assert inertia_eig(M) == prob.expected_inertia


def test_exact_singular():
    prob = mdsgen.g5_singular(200, 10, 6, 6, seed=4)
    M, _, _ = oracle.condense(prob)
    LD, ipiv, info = oracle.bk_factor(M)
    _, _, info_l = _lapack_bk(M)
    assert info > 0 and info_l > 0
    assert oracle.inertia(LD, ipiv, oracle.default_tol(M)) == prob.expected_inertia
    with pytest.raises(oracle.OracleError) as e:
        oracle.bk_solve(LD, ipiv, np.ones(M.shape[0]), oracle.default_tol(M))
    assert e.value.code == oracle.ERR_SINGULAR


@pytest.mark.parametrize("seed", range(12))
def test_solve_vs_lapack_dsytrs_and_numpy(seed):
    n = 10 + 13 * seed
    A = mdsgen.g4_random_symmetric(n, 40 + seed, shrink_diag=(seed % 2 == 1))
    b = np.random.default_rng(seed).standard_normal(n)
    LD, ipiv, _ = oracle.bk_factor(A)
    x = oracle.bk_solve(LD, ipiv, b, 0.0)
    ldu, ipiv_l, _ = _lapack_bk(A)
    x_l, info = lapack.dsytrs(ldu, ipiv_l, b, lower=1)
    As = sym_from_lower(A)
    assert rel_inf(x, x_l) <= 1e-9
    assert rel_inf(x, np.linalg.solve(As, b)) <= 1e-9


def test_solve_spec_examples_and_residual():
    # SPEC.md:217-219
    LD, ipiv, _ = oracle.bk_factor(np.eye(3))
    np.testing.assert_array_equal(oracle.bk_solve(LD, ipiv, np.array([1.0, 2.0, 3.0]), 0.0), [1, 2, 3])
    LD, ipiv, _ = oracle.bk_factor(np.diag([2.0, 4.0]))
    np.testing.assert_array_equal(oracle.bk_solve(LD, ipiv, np.array([2.0, 8.0]), 0.0), [1, 2])
    # R9: ||Kx-b||/||b|| <= 1e-12 on well-conditioned (kappa <= 1e4) inputs
    for N in (50, 150):
        A, _ = mdsgen.g3_prescribed(N, seed=3 * N)
        b = np.random.default_rng(N).standard_normal(N)
        LD, ipiv, _ = oracle.bk_factor(A)
        x = oracle.bk_solve(LD, ipiv, b, oracle.default_tol(A))
        As = sym_from_lower(A)
        assert np.linalg.cond(As) <= 1e4
        assert np.abs(As @ x - b).max() / np.abs(b).max() <= 1e-12


def test_anorm_and_nonfinite():
    A = mdsgen.g4_random_symmetric(20, 1)
    assert abs(oracle.anorm_lower(A) - np.abs(sym_from_lower(A)).sum(1).max()) <= 1e-12 * np.abs(A).sum()
    A[5, 2] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        oracle.anorm_lower(A)
    assert e.value.code == oracle.ERR_NONFINITE


def test_threaded_factor_bit_identical_and_pinned():
    # The OpenMP split of the trailing update (columns j are independent; the 2x2 step
    # keeps dsytf2's operand order) must not change a single bit, and must still be BK:
    # at N = 1400 (above the threading threshold) with many 2x2 pivots the inertia equals
    # the closed form of the prescribed-spectrum generator, the product-form factors
    # reconstruct A, and the solve meets the residual bar.
    A, ine = mdsgen.g3_prescribed(1400, seed=77, n2x2=350)
    nt = oracle.num_threads()
    try:
        oracle.set_threads(1)
        LD1, ip1, _ = oracle.bk_factor(A)
        oracle.set_threads(max(nt, 4))
        LD4, ip4, _ = oracle.bk_factor(A)
    finally:
        oracle.set_threads(nt)
    np.testing.assert_array_equal(LD1, LD4)
    np.testing.assert_array_equal(ip1, ip4)
    assert (ip1 < 0).sum() > 100                                     # the 2x2 branch ran
    assert oracle.inertia(LD1, ip1, oracle.default_tol(A)) == ine
    b = np.random.default_rng(5).standard_normal(1400)
    x = oracle.bk_solve(LD1, ip1, b, oracle.default_tol(A))
    As = sym_from_lower(A)
    assert np.abs(As @ x - b).max() / np.abs(b).max() <= 1e-12
