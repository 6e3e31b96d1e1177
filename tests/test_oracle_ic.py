"""Inertia correction: the oracle loop against the
closed forms the paper and the generators fix.
G6 puts prescribed negative eigenvalues in H_dd with weak coupling, so the
smallest acceptable delta_w is -min(lambda) up to O(jd_norm^2): the accepted
value is the first element of the IC sequence above it."""
import numpy as np
import pytest

import mdsgen
import oracle

SHAPE = dict(n_s=1500, n_d=24, m_E=8, m_I=8)


def ic_sequence(delta_w_last, n, p=oracle.IC_DEFAULTS):
    """The delta_w values IC-3/IC-5 try, written from the rule (for the pins)."""
    dw = p["delta_w0"] if delta_w_last == 0.0 else max(p["delta_w_min"], p["kappa_w_minus"] * delta_w_last)
    out = []
    for _ in range(n):
        out.append(dw)
        dw *= p["kappa_w_plus_first"] if delta_w_last == 0.0 else p["kappa_w_plus"]
    return out


def test_convex_accepted_without_regularisation():
    # SPEC.md:431 example 1: convex, strictly feasible -> delta_w = 0, inertia (n_d, 0, m), one trial
    p = mdsgen.g1_quasidefinite(**SHAPE, seed=11)
    r = oracle.inertia_correction(p, mu=0.1)
    assert r["delta_w"] == 0.0 and r["delta_c"] == 0.0 and len(r["trials"]) == 1
    assert r["inertia"] == (p.n_d, 0, p.m_E + p.m_I)


@pytest.mark.parametrize("lam_min", [-3.0, -0.03, -250.0])
def test_negative_curvature_first_sufficient_multiple(lam_min):
    # SPEC.md:432 example 2: Q_dd with a negative eigenvalue forces delta_w > 0; the accepted
    # delta_w is the first IC multiple exceeding -lambda_min (closed form for weak coupling)
    p = mdsgen.g6_negative_curvature(**SHAPE, seed=12, lam_neg=(lam_min,))
    r = oracle.inertia_correction(p, mu=0.1)
    seq = ic_sequence(0.0, 12)
    expect = next(d for d in seq if d > -lam_min)
    assert r["delta_w"] == expect and r["delta_w_last"] == expect
    assert [t[0] for t in r["trials"]] == [0.0] + seq[:seq.index(expect) + 1]
    assert r["inertia"] == (p.n_d, 0, p.m_E + p.m_I)
    # every rejected trial has exactly the closed-form inertia of H_dd + delta_w I
    lam = p.meta["lam"]
    for dw, dc, ine in r["trials"][:-1]:
        neg = int(np.sum(lam + dw < 0))
        assert ine == (p.n_d - neg, 0, p.m_E + p.m_I + neg)
    # monotone within the episode
    dws = [t[0] for t in r["trials"]]
    assert all(b > a for a, b in zip(dws, dws[1:]))


def test_warm_start_from_delta_w_last():
    # IC-3: the next episode starts at kappa_w_minus * delta_w_last and escalates by kappa_w_plus
    p = mdsgen.g6_negative_curvature(**SHAPE, seed=13, lam_neg=(-3.0,))
    r1 = oracle.inertia_correction(p, mu=0.1)
    assert r1["delta_w"] == 100.0                         # 1e-4 -> 1e-2 -> 1 -> 100
    r2 = oracle.inertia_correction(p, mu=0.1, delta_w_last=r1["delta_w_last"])
    w0 = (1.0 / 3.0) * 100.0                              # kappa_w_minus * delta_w_last
    assert [t[0] for t in r2["trials"]] == [0.0, w0]
    q = mdsgen.g6_negative_curvature(**SHAPE, seed=13, lam_neg=(-50.0,))
    r3 = oracle.inertia_correction(q, mu=0.1, delta_w_last=100.0)
    assert [t[0] for t in r3["trials"]] == [0.0, w0, 8.0 * w0]


def test_zero_eigenvalue_triggers_delta_c():
    # IC-2: an exactly singular M (G5: zero row/column) -> delta_c = delta_c_bar * mu^kappa_c,
    # which makes the zero pivot negative: accepted at the first delta_w trial
    p = mdsgen.g5_singular(**SHAPE, seed=14)
    mu = 0.01
    r = oracle.inertia_correction(p, mu=mu)
    assert r["trials"][0][2] == p.expected_inertia            # (n_d, 1, m-1)
    assert r["delta_c"] == 1e-8 * mu ** 0.25
    assert r["delta_w"] == 1e-4 and len(r["trials"]) == 2
    assert r["inertia"] == (p.n_d, 0, p.m_E + p.m_I)


def test_singular_system_when_delta_w_exceeds_max():
    p = mdsgen.g6_negative_curvature(**SHAPE, seed=15, lam_neg=(-3.0,))
    with pytest.raises(oracle.OracleError):
        oracle.inertia_correction(p, mu=0.1, params=dict(delta_w_max=2.0))


def test_accepted_step_solves_the_regularised_system():
    # the returned direction solves Eq.(5) with +delta_w on Q_xs, Q_xd (and -delta_c on the
    # constraint blocks): dense brute force of the full (n_s+N) system
    import dataclasses
    p = mdsgen.g6_negative_curvature(n_s=300, n_d=12, m_E=4, m_I=4, seed=16, lam_neg=(-2.0,))
    r = oracle.inertia_correction(p, mu=0.1)
    q = dataclasses.replace(p, delta_w=r["delta_w"], delta_c=r["delta_c"])
    n_s, n_d, m = q.n_s, q.n_d, q.m_E + q.m_I
    Js = np.zeros((n_s, m))
    for k in range(n_s):
        for t in range(q.rowptr[k], q.rowptr[k + 1]):
            Js[k, q.colidx[t]] = q.val[t]
    Hd = np.asarray(q.H_dd)
    Hd = np.tril(Hd) + np.tril(Hd, -1).T
    Nf = n_s + n_d + m
    K = np.zeros((Nf, Nf))
    K[:n_s, :n_s] = np.diag(q.h_ss + q.sigma_s + q.delta_w)
    K[n_s:n_s + n_d, n_s:n_s + n_d] = Hd + np.diag(q.sigma_d + q.delta_w)
    K[n_s + n_d:, :n_s] = Js.T
    K[:n_s, n_s + n_d:] = Js
    K[n_s + n_d:, n_s:n_s + n_d] = np.asarray(q.J_d)
    K[n_s:n_s + n_d, n_s + n_d:] = np.asarray(q.J_d).T
    Dyy = np.concatenate([np.zeros(q.m_E), 1.0 / np.asarray(q.d_h)]) + q.delta_c
    K[n_s + n_d:, n_s + n_d:] = -np.diag(Dyy)
    x = np.linalg.solve(K, np.asarray(q.r))
    got = np.concatenate([r["dx_s"], r["dxy"]])
    assert np.abs(got - x).max() <= 1e-10 * np.abs(x).max()
