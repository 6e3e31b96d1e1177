"""Pins for oracle O7 (barrier vector kernels, K1; fraction-to-boundary
PAPER.md:140): SPEC examples, a brute-force
alpha scan + maximality, and closed-form sums."""
import numpy as np
import pytest

import mdsgen
import oracle
from tests.helpers import golden


def _sv(x, dx, lo, up, zl=None, zu=None, dzl=None, dzu=None, tau=0.99, mu=0.0):
    n = len(x)
    z = np.ones(n)
    zl = z if zl is None else zl
    zu = z if zu is None else zu
    dzl = np.zeros(n) if dzl is None else dzl
    dzu = np.zeros(n) if dzu is None else dzu
    return oracle.step_vectors(np.array(x, float), np.array(dx, float), np.array(lo, float), np.array(up, float),
                               np.array(zl, float), np.array(zu, float), np.array(dzl, float), np.array(dzu, float),
                               tau, mu)


def test_alpha_spec_examples():
    g = golden("step_examples.json")
    for c in g["alpha_cases"]:
        st, res, _ = _sv(c["x"], c["dx"], c["lo"], c["up"], tau=c["tau"])
        assert st == oracle.OK
        assert abs(res["alpha_p"] - c["alpha"]) <= 1e-15


def test_sigma_and_complementarity_examples():
    g = golden("step_examples.json")
    for c in g["sigma_cases"]:
        st, res, sig = _sv(c["x"], [0.0], c["lo"], c["up"], zl=c["zl"], zu=c["zu"])
        assert sig[0] == c["sigma"][0]
    c = g["compl_case"]
    st, res, _ = _sv(c["x"], [0.0], c["lo"], c["up"], zl=c["zl"], zu=c["zu"], mu=c["mu"])
    assert res["compl_inf"] == c["compl_inf"]


@pytest.mark.parametrize("seed", range(8))
def test_alpha_bruteforce_scan_and_maximality(seed):
    sv = mdsgen.step_vectors(40, seed)
    st, res, _ = oracle.step_vectors(sv.x, sv.dx, sv.lo, sv.up, sv.zl, sv.zu, sv.dzl, sv.dzu, sv.tau, sv.mu)
    assert st == oracle.OK
    a = res["alpha_p"]
    fin_lo = np.abs(sv.lo) < mdsgen.INF
    fin_up = np.abs(sv.up) < mdsgen.INF

    def ok(al):
        xn = sv.x + al * sv.dx
        c1 = np.all((xn - sv.lo >= (1 - sv.tau) * (sv.x - sv.lo) * (1 - 1e-12))[fin_lo])
        c2 = np.all((sv.up - xn >= (1 - sv.tau) * (sv.up - sv.x) * (1 - 1e-12))[fin_up])
        return c1 and c2
    assert ok(a)
    if a < 1.0:
        assert not ok(a * (1 + 1e-9))
    grid = np.linspace(0, 1, 20001)
    feas = [al for al in grid if ok(al)]
    assert abs(max(feas) - a) <= 1e-4
    # dual step: same rule on z >= (1-tau) z
    ad = res["alpha_d"]
    zl_new = sv.zl + ad * sv.dzl
    zu_new = sv.zu + ad * sv.dzu
    assert np.all((zl_new >= (1 - sv.tau) * sv.zl * (1 - 1e-12))[fin_lo])
    assert np.all((zu_new >= (1 - sv.tau) * sv.zu * (1 - 1e-12))[fin_up])


def test_sums_and_sigma_closed_form():
    sv = mdsgen.step_vectors(1000, 3, mu=0.05)
    st, res, sig = oracle.step_vectors(sv.x, sv.dx, sv.lo, sv.up, sv.zl, sv.zu, sv.dzl, sv.dzu, sv.tau, sv.mu)
    fl = np.abs(sv.lo) < mdsgen.INF
    fu = np.abs(sv.up) < mdsgen.INF
    cl = (sv.x - sv.lo) * sv.zl
    cu = (sv.up - sv.x) * sv.zu
    assert res["n_compl"] == fl.sum() + fu.sum()
    assert abs(res["compl_sum"] - (cl[fl].sum() + cu[fu].sum())) <= 1e-12 * res["compl_sum"]
    assert res["compl_inf"] == max(np.abs(cl[fl] - sv.mu).max(), np.abs(cu[fu] - sv.mu).max())
    exp = np.where(fl, sv.zl / np.where(fl, sv.x - sv.lo, 1), 0) + np.where(fu, sv.zu / np.where(fu, sv.up - sv.x, 1), 0)
    assert np.abs(sig - exp).max() <= 1e-15 * np.abs(exp).max()


def test_not_interior():
    st, res, _ = _sv([0.0, 1.0], [0.0, 0.0], [0.0, -1e20], [1.0, 1e20])
    assert st == oracle.ERR_NOT_INTERIOR and res["first_bad"] == 0
    st, res, _ = _sv([0.5, 0.5], [0.0, 0.0], [0.0, 0.0], [1.0, 1.0], zl=[1.0, -1.0], zu=[1.0, 1.0])
    assert st == oracle.ERR_NOT_INTERIOR and res["first_bad"] == 1


def test_norm_inf():
    # SPEC.md:84 INF_NORM of zeros -> 0; |.|max
    assert oracle.norm_inf(np.zeros(3)) == 0.0
    assert oracle.norm_inf(np.array([3.0, -4.0])) == 4.0
