"""Pins of the oracle's interior-point loop (oracle/ipm.py, R23) to
what the mathematics fixes, independently of the oracle's own arithmetic:
  * separable box QP  min 1/2 h x^2 + c x on [lo, up]: x* = clip(-c/h, lo, up) (closed form);
  * equality-constrained QP without bounds: the dense KKT system [[H, J^T], [J, 0]] solved by numpy;
  * general convex QP: the KKT conditions hold at the returned point, checked on a dense
    assembly of H and J (not the oracle's mat-vec), and x equals the solution of the
    equality-constrained QP on the active set the IPM identified (dense numpy solve);
  * SPEC.md:450-452 barrier-update example (mu 0.1 -> 0.02)."""
import dataclasses

import numpy as np
import pytest

import mdsgen
from oracle import ipm
from tests.helpers import dense_qp_parts as dense_parts

INF = 1e20


def test_separable_box_qp_closed_form():
    qp = mdsgen.qp_problem(300, 4, 2, 2, seed=5, box_frac=1.0)
    b = qp.base
    # drop every coupling: m = 0, n_d dense block kept diagonal
    base = dataclasses.replace(b, m_E=0, m_I=0, rowptr=np.arange(b.n_s + 1, dtype=np.int32) * 0,
                               colidx=np.zeros(0, dtype=np.int32), val=np.zeros(0), J_d=np.zeros((0, b.n_d), order="F"),
                               d_h=np.zeros(0), H_dd=np.asfortranarray(np.diag(np.linspace(0.5, 2.0, b.n_d))))
    rng = np.random.default_rng(1)
    c = rng.standard_normal(b.n_s + b.n_d) * 8.0           # some optima on the box faces
    q = mdsgen.QPProblem(base, c, np.zeros(0), np.zeros(0), np.zeros(0), qp.lo, qp.up, qp.x_star)
    res = ipm.solve(q)
    assert res["status"] == "Optimal"
    h = np.concatenate([base.h_ss, np.diag(np.asarray(base.H_dd))])
    x_exact = np.clip(-c / h, qp.lo, qp.up)
    # an interior point stops with gap * z <= tol: an active variable sits tol / z from its bound
    assert np.abs(res["x"] - x_exact).max() <= 1e-6
    assert (np.abs(x_exact) == 10.0).any() and (np.abs(x_exact) < 10.0).any()


def test_equality_qp_dense_kkt():
    qp = mdsgen.qp_problem(2000, 30, 25, 0, seed=9, box_frac=0.0)
    res = ipm.solve(qp)
    assert res["status"] == "Optimal"
    H, J = dense_parts(qp)
    n, m = H.shape[0], J.shape[0]
    K = np.block([[H, J.T], [J, np.zeros((m, m))]])
    sol = np.linalg.solve(K, np.concatenate([-qp.c, qp.g_E]))
    assert np.abs(res["x"] - sol[:n]).max() <= 1e-8 * max(1.0, np.abs(sol[:n]).max())
    assert np.abs(res["y"] - sol[n:]).max() <= 1e-6 * max(1.0, np.abs(sol[n:]).max())


@pytest.mark.parametrize("shape,seed,pattern", [((400, 20, 10, 10), 1, "uniform"), ((3000, 60, 30, 40), 2, "local"),
                                                ((5000, 80, 0, 50), 3, "uniform")])
def test_general_qp_kkt_and_active_set(shape, seed, pattern):
    qp = mdsgen.qp_problem(*shape, seed=seed, pattern=pattern)
    res = ipm.solve(qp)
    assert res["status"] == "Optimal" and res["e0"] <= 1e-8
    H, J = dense_parts(qp)
    b = qp.base
    m_E = b.m_E
    x, s, y = res["x"], res["s"], res["y"]
    zl, zu, vl, vu = res["zl"], res["zu"], res["vl"], res["vu"]
    # KKT of the convex QP (sufficient for global optimality)
    assert np.abs(H @ x + qp.c + J.T @ y - zl + zu).max() <= 1e-7
    assert np.abs(J[:m_E] @ x - qp.g_E).max(initial=0.0) <= 1e-7
    assert np.abs(J[m_E:] @ x - s).max() <= 1e-7
    assert np.abs(-y[m_E:] - vl + vu).max() <= 1e-7
    fl, fu = qp.lo > -INF, qp.up < INF
    assert (x[fl] > qp.lo[fl]).all() and (x[fu] < qp.up[fu]).all()
    assert (s > qp.h_l).all() and (s < qp.h_u).all()
    assert (zl >= 0).all() and (zu >= 0).all() and (vl >= 0).all() and (vu >= 0).all()
    assert (np.abs((x - qp.lo)[fl] * zl[fl]).max(initial=0) <= 1e-8)
    # the active set the duals identify -> equality-constrained QP, dense solve
    act_lo = fl & (zl > 1e-5)
    act_up = fu & (zu > 1e-5)
    act_hl, act_hu = vl > 1e-5, vu > 1e-5
    n = H.shape[0]
    rows = [J[:m_E]]
    rhs = [qp.g_E]
    for mask, val in ((act_lo, qp.lo), (act_up, qp.up)):
        E = np.eye(n)[mask]
        rows.append(E)
        rhs.append(val[mask])
    for mask, val in ((act_hl, qp.h_l), (act_hu, qp.h_u)):
        rows.append(J[m_E:][mask])
        rhs.append(val[mask])
    A = np.vstack(rows)
    K = np.block([[H, A.T], [A, np.zeros((A.shape[0], A.shape[0]))]])
    sol = np.linalg.lstsq(K, np.concatenate([-qp.c, np.concatenate(rhs)]), rcond=None)[0]
    assert np.abs(x - sol[:n]).max() <= 1e-6 * max(1.0, np.abs(sol[:n]).max())


def test_barrier_update_spec_example():
    o = ipm.OPTS
    mu = 0.1
    new = max(1e-6 / 10.0, min(o["kappa_mu"] * mu, mu ** o["theta_mu"]))   # SPEC.md:451 (tol = 1e-6)
    assert new == pytest.approx(0.02)


def test_nlpmds_ex4_structure():
    # PAPER.md:536 / SPEC.md:288-297: n_d = n_s = k, m = n_s + 3, compressed size 2k + 3
    for k in (1, 10, 100):
        q = mdsgen.synthetic_problem(k)
        b = q.base
        assert b.n_d == b.n_s == k and b.m == k + 3 and b.N == 2 * k + 3


@pytest.mark.parametrize("k", [2, 10, 100])
def test_nlpmds_ex4_closed_form_optimum(k):
    # closed form: x_d's unconstrained minimiser solves (I + ee^T/k) x_d = e -> x_d = e/2, which meets
    # the active bound mean(x_d) >= 1/2 with multiplier k/2 > 0; the first equality then forces
    # mean(x_s) = 1/2 and stationarity in x_s (x_s - 1 + y0/k = 0 with y0 = k/2) gives x_s = e/2
    q = mdsgen.synthetic_problem(k)
    res = ipm.solve(q)
    assert res["status"] == "Optimal"
    assert np.abs(res["x"] - 0.5).max() <= 1e-7
