"""Inertia correction of a scenario batch on the device (BatchedKKTStep.factor_ic:
mds_ic_begin_batched / masked mds_condense_batched + mds_factor_batched /
mds_ic_step_batched, as a host loop or as one CUDA graph with a conditional WHILE
node) against the oracle's Algorithm IC loop (oracle.inertia_correction,
PAPER.md:161; R22), scenario by scenario:
  number of trials, accepted (delta_w, delta_c) and inertia exact (the same IC
  arithmetic in FP64 on both sides), direction within 1e-8;
and the batch invariants: scenarios that need no correction are factored once,
a data error / a singular scenario is isolated, warm start carries delta_w_last."""
import numpy as np
import pytest

import mdsgen
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2605_13736_b200 as mds  # noqa: E402

SHAPE = dict(n_s=1500, n_d=40, m_E=8, m_I=12)
# one pattern (g1 seed) for the whole batch; the dense Hessians differ per scenario
LAMS = [(), (-3.0,), (-0.03, -0.02), (-250.0,), (), (-1.2e4,), (-3.0,), (-0.5,)]
# (every accepted delta_w clears -min(lambda) by a wide margin: no decision sits on the
#  O(jd_norm^2) crossover where rounding order could flip an inertia count)


def batch(lams, seed=31):
    return [mdsgen.g6_negative_curvature(**SHAPE, seed=seed, lam_neg=lam) for lam in lams]


def check(bt, probs, mu, warm=None, skip=()):
    phase, ntrial, dw, dc = bt.ic_results()
    refs = []
    for i, p in enumerate(probs):
        if i in skip:
            refs.append(None)
            continue
        ref = oracle.inertia_correction(p, mu, delta_w_last=0.0 if warm is None else warm[i])
        refs.append(ref)
        assert phase[i] == 2, (i, phase[i])
        assert ntrial[i] == len(ref["trials"]), (i, ntrial[i], ref["trials"])
        assert dw[i] == ref["delta_w"], (i, dw[i], ref["delta_w"])
        # delta_c = delta_c_bar * mu^kappa_c: CUDA pow and libm pow may differ in the last ulp
        assert abs(dc[i] - ref["delta_c"]) <= 4e-16 * ref["delta_c"], (i, dc[i], ref["delta_c"])
        out = bt.results(i)
        assert out["status"] == 0
        assert out["inertia"] == ref["inertia"] == (p.n_d, 0, p.m_E + p.m_I)
        assert np.abs(out["dxy"] - ref["dxy"]).max() <= 1e-8 * np.abs(ref["dxy"]).max()
        assert np.abs(out["dx_s"] - ref["dx_s"]).max() <= 1e-8 * np.abs(ref["dx_s"]).max()
    return refs


@pytest.mark.parametrize("mode", ["graph", "host"])
def test_batched_ic_matches_oracle(mode):
    probs = batch(LAMS)
    bt = mds.BatchedKKTStep(probs)
    bt.factor_ic(0.05, mode=mode)
    bt.finish()
    refs = check(bt, probs, 0.05)
    # the trial counts differ across the batch: the mask really was exercised
    assert len({len(r["trials"]) for r in refs}) >= 3
    # warm start: delta_w_last persists on the device; a second call follows the
    # oracle started from the first call's accepted delta_w
    warm = [r["delta_w_last"] for r in refs]
    bt.factor_ic(0.05, mode=mode)
    bt.finish()
    check(bt, probs, 0.05, warm=warm)


def test_batched_ic_graph_equals_host_loop_bitwise():
    probs = batch(LAMS[:5], seed=32)
    a, b = mds.BatchedKKTStep(probs), mds.BatchedKKTStep(probs)
    a.factor_ic(0.1, mode="graph")
    a.finish()
    b.factor_ic(0.1, mode="host")
    b.finish()
    for i in range(len(probs)):
        ra, rb = a.results(i), b.results(i)
        np.testing.assert_array_equal(ra["dxy"], rb["dxy"])
        np.testing.assert_array_equal(ra["dx_s"], rb["dx_s"])
    for x, y in zip(a.ic_results(), b.ic_results()):
        np.testing.assert_array_equal(x, y)


def test_batched_ic_result_independent_of_batch():
    # a scenario's correction and direction do not depend on its neighbours' trials
    probs = batch(LAMS, seed=33)
    big = mds.BatchedKKTStep(probs)
    big.factor_ic(0.05)
    big.finish()
    for i in (1, 3):
        one = mds.BatchedKKTStep([probs[i]], plan=big.plan)
        one.factor_ic(0.05)
        one.finish()
        np.testing.assert_array_equal(one.results(0)["dxy"], big.results(i)["dxy"])
        assert one.ic_results()[1][0] == big.ic_results()[1][i]


def test_batched_ic_isolates_errors_and_singular():
    probs = batch([(), (-3.0,), (-250.0,), (-3.0,)], seed=34)
    bad = probs[3]
    bad.H_dd = np.array(bad.H_dd, order="F", copy=True)
    bad.H_dd[5, 2] = np.nan                                   # (lower triangle) data error: phase 4, no escalation
    bt = mds.BatchedKKTStep(probs)
    # delta_w runs 1e-4, 1e-2, 1, 100, 1e4 (kappa_w_plus_first = 100 while delta_w_last = 0):
    # with delta_w_max = 500 scenario 1 (lambda = -3) is accepted at 100, scenario 2
    # (lambda = -250) fails (singular)
    bt._ic_setup(mds.ICParams(delta_w_max=500.0))
    bt.factor_ic(0.05)
    bt.finish()
    phase, ntrial, dw, dc = bt.ic_results()
    st = bt.status.cpu().numpy()
    assert phase[3] == 4 and ntrial[3] == 1 and st[3] == mds.NumericError.code
    assert phase[2] == 3 and st[2] == mds.SingularError.code
    with pytest.raises(oracle.OracleError):
        oracle.inertia_correction(probs[2], 0.05, params=dict(delta_w_max=500.0))
    ref = oracle.inertia_correction(probs[1], 0.05, params=dict(delta_w_max=500.0))
    assert phase[1] == 2 and ntrial[1] == len(ref["trials"]) and dw[1] == ref["delta_w"]
    assert phase[0] == 2 and ntrial[0] == 1 and dw[0] == 0.0
    for i in (0, 1):
        r = oracle.inertia_correction(probs[i], 0.05, params=dict(delta_w_max=500.0))
        out = bt.results(i)
        assert out["status"] == 0
        assert np.abs(out["dxy"] - r["dxy"]).max() <= 1e-8 * np.abs(r["dxy"]).max()


def test_batched_ic_zero_eigenvalue_sets_delta_c():
    # G5 (exactly singular M: zero row) -> IC-2 sets delta_c = delta_c_bar mu^kappa_c; every
    # scenario shares the G5 pattern, Hessians shifted so the trial counts differ
    base = mdsgen.g5_singular(**SHAPE, seed=35)
    probs = []
    for shift in (0.0, -4.0, -40.0):
        p = mdsgen.g5_singular(**SHAPE, seed=35)
        p.H_dd = np.asfortranarray(np.asarray(base.H_dd) + shift * np.eye(SHAPE["n_d"]))
        probs.append(p)
    bt = mds.BatchedKKTStep(probs)
    bt.factor_ic(0.02)
    bt.finish()
    refs = check(bt, probs, 0.02)
    assert all(r["delta_c"] > 0 for r in refs)
