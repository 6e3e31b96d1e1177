"""Pins for oracle O1 (condensation, Eq.(5)->Eq.(6)) and O6 (sparse-step
recovery).  Each pin is independent of the oracle's own arithmetic: the SPEC
worked example, a hand-derived integer solution, a dense brute-force
materialisation, the full 4x4 system solved by numpy, a special case and a
mutation test."""
import numpy as np
import pytest

import mdsgen
import oracle
from tests.helpers import dense_js, full_kkt4, golden, inertia_eig, rel_inf, sym_from_lower


def worked_problem():
    g = golden("worked_example.json")
    rowptr = np.array([0, 2], dtype=np.int32)
    colidx = np.array(g["J_s_row0"]["cols"], dtype=np.int32)
    val = np.array(g["J_s_row0"]["vals"])
    return mdsgen.MDSProblem(
        n_s=1, n_d=1, m_E=1, m_I=1, rowptr=rowptr, colidx=colidx, val=val,
        h_ss=np.array([g["q_ss"]]), sigma_s=np.array([0.0]),
        H_dd=np.asfortranarray([[g["Q_d"]]]), sigma_d=np.array([0.0]),
        J_d=np.asfortranarray(g["J_d"]), d_h=np.array(g["d_h"]), r=np.array(g["r"]))


def test_worked_example_matrix():
    g = golden("worked_example.json")
    prob = worked_problem()
    M, rhs, w = oracle.condense(prob)
    np.testing.assert_array_equal(np.tril(M), np.tril(np.array(g["M"])))
    assert w[0] == 0.5
    # full 4x4 matrix of the golden file equals the test-side Eq.(5) assembly
    np.testing.assert_array_equal(full_kkt4(prob), np.array(g["K4"], dtype=float))


def test_worked_example_solution_and_inertia():
    g = golden("worked_example.json")
    prob = worked_problem()
    out = oracle.newton_step(prob)
    sol = np.array(g["solution"])
    np.testing.assert_allclose(out["dx_s"], sol[:1], rtol=0, atol=1e-15)
    np.testing.assert_allclose(out["dxy"], sol[1:], rtol=0, atol=1e-15)
    assert out["inertia"] == tuple(g["inertia_M"])
    # Haynsworth: inertia(K4) = inertia(Q_s) + inertia(M)
    ine = out["inertia"]
    assert (ine[0] + prob.n_s, ine[1], ine[2]) == tuple(g["inertia_K4"])


def test_dimension_reduction_by_ns():
    # PAPER.md:178 "The reduction offered by the above system is n_s"
    prob = mdsgen.g1_quasidefinite(50, 6, 3, 4, seed=3)
    M, _, _ = oracle.condense(prob)
    assert M.shape[0] == full_kkt4(prob).shape[0] - prob.n_s


@pytest.mark.parametrize("seed,pattern,dw,dc", [(1, "uniform", 0.0, 0.0), (2, "local", 0.3, 1e-8),
                                                 (3, "uniform", 1e-4, 0.5), (4, "local", 0.0, 0.0)])
def test_brute_force_dense_materialisation(seed, pattern, dw, dc):
    # fused M := M + A D B^T equals the dense materialisation within 1e-13
    prob = mdsgen.g1_quasidefinite(120, 7, 5, 6, seed=seed, pattern=pattern, delta_w=dw, delta_c=dc)
    M, rhs, w = oracle.condense(prob)
    J = dense_js(prob)
    q = prob.h_ss + prob.sigma_s + dw
    Wd = 1.0 / q
    yy = -(J.T * Wd) @ J - dc * np.eye(prob.m)
    yy[prob.m_E:, prob.m_E:] -= np.diag(1.0 / prob.d_h)
    n_d = prob.n_d
    H = sym_from_lower(prob.H_dd) + np.diag(prob.sigma_d) + dw * np.eye(n_d)
    Mref = np.block([[H, np.asarray(prob.J_d).T], [np.asarray(prob.J_d), yy]])
    assert rel_inf(np.tril(M), np.tril(Mref)) <= 1e-13
    np.testing.assert_allclose(w, Wd, rtol=0, atol=0)
    r = prob.r
    rhs_ref = np.concatenate([r[prob.n_s:prob.n_s + n_d], r[prob.n_s + n_d:] - J.T @ (Wd * r[:prob.n_s])])
    assert rel_inf(rhs, rhs_ref) <= 1e-13


@pytest.mark.parametrize("seed", range(6))
def test_compression_equivalence_full_system(seed):
    # condensed solve + recovery == dense solve of Eq.(5), rel <= 1e-8
    pattern = "uniform" if seed % 2 else "local"
    prob = mdsgen.g1_quasidefinite(200 + 37 * seed, 9, 4, 7, seed=100 + seed, pattern=pattern,
                                   delta_w=0.01 * seed, delta_c=1e-8 * seed)
    K = full_kkt4(prob)
    x_full = np.linalg.solve(K, prob.r)
    out = oracle.newton_step(prob)
    x_c = np.concatenate([out["dx_s"], out["dxy"]])
    assert rel_inf(x_c, x_full) <= 1e-10
    # and the condensed solve's own residual on K4 (R9)
    assert np.abs(K @ x_c - prob.r).max() / np.abs(prob.r).max() <= 1e-12
    # Haynsworth: inertia(K4) = (n_s,0,0) + inertia(M), K4 inertia by eigvalsh
    ik = inertia_eig(K)
    im = out["inertia"]
    assert ik == (im[0] + prob.n_s, im[1], im[2])
    assert im == prob.expected_inertia


def test_no_sparse_coupling_special_case():
    # J_s = 0 -> M_yy = -diag(0, 1/d_h) - delta_c I
    prob = mdsgen.g1_quasidefinite(30, 4, 3, 2, seed=9, delta_c=0.25)
    prob.val = np.zeros_like(prob.val)
    M, _, _ = oracle.condense(prob)
    yy = M[prob.n_d:, prob.n_d:]
    exp = -0.25 * np.eye(prob.m)
    exp[prob.m_E:, prob.m_E:] -= np.diag(1.0 / prob.d_h)
    np.testing.assert_array_equal(np.tril(yy), np.tril(exp))


def test_recover_special_cases():
    # J_s = 0 -> dx_s = r_xs / q ; r_xs = 0, dy = 0 -> 0
    prob = mdsgen.g1_quasidefinite(40, 3, 2, 2, seed=5)
    q = prob.h_ss + prob.sigma_s
    w = 1.0 / q
    r_xs = prob.r[:prob.n_s]
    z = prob.val.copy()
    prob.val = np.zeros_like(z)
    dx = oracle.recover(prob, w, r_xs, np.ones(prob.m))
    np.testing.assert_array_equal(dx, w * r_xs)
    prob.val = z
    dx0 = oracle.recover(prob, w, np.zeros(prob.n_s), np.zeros(prob.m))
    assert np.all(dx0 == 0.0)
    # brute force: w .* (r - J dy)
    dy = np.random.default_rng(0).standard_normal(prob.m)
    dx = oracle.recover(prob, w, r_xs, dy)
    assert rel_inf(dx, w * (r_xs - dense_js(prob) @ dy)) <= 1e-15


def test_mutation_sign_flip_is_caught():
    # a sign flip in the K3 term must fail the equivalence suite
    prob = mdsgen.g1_quasidefinite(150, 6, 4, 4, seed=21)
    M, rhs, w = oracle.condense(prob)
    J = dense_js(prob)
    Mbad = np.array(M)
    Mbad[prob.n_d:, prob.n_d:] += 2.0 * np.tril((J.T * w) @ J)   # flips the sign of -J^T W J
    LD, ipiv, _ = oracle.bk_factor(Mbad)
    dxy = oracle.bk_solve(LD, ipiv, rhs, 0.0)
    dxs = oracle.recover(prob, w, prob.r[:prob.n_s], dxy[prob.n_d:])
    x_full = np.linalg.solve(full_kkt4(prob), prob.r)
    assert rel_inf(np.concatenate([dxs, dxy]), x_full) > 1e-3


def test_errors():
    prob = mdsgen.g1_quasidefinite(20, 3, 2, 2, seed=1)
    bad = mdsgen.g1_quasidefinite(20, 3, 2, 2, seed=1)
    bad.h_ss = bad.h_ss.copy(); bad.sigma_s = bad.sigma_s.copy()
    bad.h_ss[3] = -5.0
    with pytest.raises(oracle.OracleError) as e:
        oracle.condense(bad)
    assert e.value.code == oracle.ERR_NONPOSITIVE
    unsorted = mdsgen.g1_quasidefinite(20, 3, 2, 2, seed=1)
    k = int(np.argmax(np.diff(unsorted.rowptr) >= 2))
    p = unsorted.rowptr[k]
    unsorted.colidx = unsorted.colidx.copy()
    unsorted.colidx[p], unsorted.colidx[p + 1] = unsorted.colidx[p + 1], unsorted.colidx[p]
    with pytest.raises(oracle.OracleError) as e:
        oracle.condense(unsorted)
    assert e.value.code == oracle.ERR_PATTERN
    dh = mdsgen.g1_quasidefinite(20, 3, 2, 2, seed=1)
    dh.d_h = np.zeros(2)
    with pytest.raises(oracle.OracleError):
        oracle.condense(dh)
    oracle.condense(prob)


def test_empty_blocks():
    # zero-length edge cases (PAPER.md:511 zero-length copies): n_s=0, m_I=0, m_E=0
    for shp in [(0, 4, 2, 3), (10, 4, 3, 0), (10, 4, 0, 3), (10, 0, 3, 3)]:
        prob = mdsgen.g1_quasidefinite(*shp, seed=2)
        out = oracle.newton_step(prob)
        K = full_kkt4(prob)
        x = np.concatenate([out["dx_s"], out["dxy"]])
        assert np.abs(K @ x - prob.r).max() <= 1e-12 * max(1, np.abs(prob.r).max())
