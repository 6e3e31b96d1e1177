"""Inertia correction through the CUDA path (paper_2605_13736_b200.InertiaCorrection:
mds_condense + mds_factor per trial, 24-byte inertia to the host) against the oracle
loop: the same trial sequence (delta_w, delta_c, inertia -- integers and exactly the
same IC arithmetic), and the accepted direction within the north-star tolerance."""
import numpy as np
import pytest

import mdsgen
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2605_13736_b200 as mds  # noqa: E402

SHAPE = dict(n_s=1500, n_d=24, m_E=8, m_I=8)


def run_both(p, mu, warm=None):
    st = mds.KKTStep(mds.DeviceProblem(p))
    ic = mds.InertiaCorrection(st)
    ref = None
    if warm is not None:
        ic.delta_w_last = warm
    g = ic.solve(mu)
    out = st.results()
    ref = oracle.inertia_correction(p, mu, delta_w_last=warm or 0.0)
    return g, out, ref, ic


@pytest.mark.parametrize("case", ["convex", "neg3", "neg_small", "neg_large", "singular"])
def test_ic_matches_oracle(case):
    gen = {"convex": lambda: mdsgen.g1_quasidefinite(**SHAPE, seed=21),
           "neg3": lambda: mdsgen.g6_negative_curvature(**SHAPE, seed=22, lam_neg=(-3.0,)),
           "neg_small": lambda: mdsgen.g6_negative_curvature(**SHAPE, seed=23, lam_neg=(-0.03, -0.02)),
           "neg_large": lambda: mdsgen.g6_negative_curvature(**SHAPE, seed=24, lam_neg=(-250.0,)),
           "singular": lambda: mdsgen.g5_singular(**SHAPE, seed=25)}[case]
    p = gen()
    g, out, ref, ic = run_both(p, mu=0.05)
    assert g["trials"] == ref["trials"]
    assert (g["delta_w"], g["delta_c"], g["inertia"]) == (ref["delta_w"], ref["delta_c"], ref["inertia"])
    assert out["status"] == 0 and out["inertia"] == (p.n_d, 0, p.m_E + p.m_I)
    assert np.abs(out["dxy"] - ref["dxy"]).max() <= 1e-8 * np.abs(ref["dxy"]).max()
    assert np.abs(out["dx_s"] - ref["dx_s"]).max() <= 1e-8 * np.abs(ref["dx_s"]).max()


def test_ic_warm_start_matches_oracle():
    p = mdsgen.g6_negative_curvature(**SHAPE, seed=26, lam_neg=(-50.0,))
    g, out, ref, ic = run_both(p, mu=0.1, warm=100.0)
    assert g["trials"] == ref["trials"] and ic.delta_w_last == ref["delta_w_last"]


def test_ic_singular_system_raises():
    p = mdsgen.g6_negative_curvature(**SHAPE, seed=27, lam_neg=(-3.0,))
    st = mds.KKTStep(mds.DeviceProblem(p))
    ic = mds.InertiaCorrection(st, mds.ICParams(delta_w_max=2.0))
    with pytest.raises(mds.SingularError):
        ic.solve(0.1)
