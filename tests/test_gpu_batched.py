"""Batched C-ABI (mds_condense_batched / mds_factor_batched / mds_solve_batched /
ipm_step_vectors_batched; SURVEY §8(b) "_batched", SCOPF scenario batches of
PAPER.md:70-78) against the CPU oracle, scenario by scenario:
  inertia exact, x and dx_s within 1e-8, rhs_c within 1e-14, w bit-exact,
  alpha / compl_inf bit-exact on the batch's own direction;
and the batch invariants: a scenario's results do not depend on the batch it
is in (bitwise), and one failing scenario does not affect the others."""
import numpy as np
import pytest

import mdsgen
import oracle
from tests.helpers import rel_inf

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2605_13736_b200 as mds  # noqa: E402


def scen(base, ids, seed):
    probs = [mdsgen.scopf_scenario(base, s, seed=seed) for s in ids]
    svs = [mdsgen.step_vectors_for(p, seed=100 + s) for p, s in zip(probs, ids)]
    return probs, svs


def check_vs_oracle(bt, i, p, sv):
    out = bt.results(i)
    ref = oracle.newton_step(p)
    assert out["status"] == 0, out["status"]
    assert out["inertia"] == ref["inertia"]
    if p.expected_inertia is not None:
        assert out["inertia"] == p.expected_inertia
    np.testing.assert_array_equal(out["w"], ref["w"])
    assert rel_inf(out["rhs_c"], ref["rhs_c"]) <= 1e-14
    assert rel_inf(out["dxy"], ref["dxy"]) <= 1e-8, rel_inf(out["dxy"], ref["dxy"])
    if p.n_s:
        assert rel_inf(out["dx_s"], ref["dx_s"]) <= 1e-8
    assert abs(out["anorm"] - oracle.anorm_lower(ref["M"])) <= 1e-13 * oracle.anorm_lower(ref["M"])
    dx = np.concatenate([out["dx_s"], out["dxy"][:p.n_d]])
    _, v, sig = oracle.step_vectors(sv.x, dx, sv.lo, sv.up, sv.zl, sv.zu, sv.dzl, sv.dzu, sv.tau, sv.mu)
    assert out["vec"]["alpha_p"] == v["alpha_p"] and out["vec"]["alpha_d"] == v["alpha_d"]
    assert out["vec"]["compl_inf"] == v["compl_inf"]
    np.testing.assert_array_equal(out["sigma"], sig)
    return out


@pytest.mark.parametrize("shape,B", [((6000, 100, 40, 60), 5), ((3000, 37, 20, 30), 3), ((20000, 300, 0, 211), 4)])
def test_batched_step_vs_oracle(shape, B):
    base = mdsgen.scopf_base(seed=7, n_s=shape[0], n_d=shape[1], m_E=shape[2], m_I=shape[3])
    probs, svs = scen(base, range(B), seed=7)
    bt = mds.BatchedKKTStep(probs, svs=svs)
    for _ in range(2):   # workspaces reusable
        bt.run()
    for i in range(B):
        check_vs_oracle(bt, i, probs[i], svs[i])


def test_batched_results_independent_of_batch():
    base = mdsgen.scopf_base(seed=8, n_s=8000, n_d=150, m_E=60, m_I=90)
    probs, svs = scen(base, range(6), seed=8)
    big = mds.BatchedKKTStep(probs, svs=svs)
    g = big.capture()
    g.replay()
    for i in (0, 4):
        one = mds.BatchedKKTStep([probs[i]], plan=big.plan, svs=[svs[i]])
        one.run()
        a, b = one.results(0), big.results(i)
        np.testing.assert_array_equal(a["dxy"], b["dxy"])
        np.testing.assert_array_equal(a["dx_s"], b["dx_s"])
        assert a["inertia"] == b["inertia"]


def test_batched_failing_scenario_is_isolated():
    base = mdsgen.scopf_base(seed=9, n_s=5000, n_d=80, m_E=30, m_I=40)
    probs, svs = scen(base, range(4), seed=9)
    bad = probs[2]
    bad.H_dd = np.array(bad.H_dd, order="F", copy=True)
    bad.H_dd[3, 1] = np.nan
    neg = probs[1]
    neg.h_ss = neg.h_ss.copy()
    neg.h_ss[10] = -50.0                          # q <= 0 -> NONPOSITIVE in scenario 1 only
    bt = mds.BatchedKKTStep(probs, svs=svs)
    bt.run()
    torch.cuda.synchronize()
    st = bt.status.cpu().numpy()
    assert st[2] == mds.NumericError.code
    assert st[1] == mds.CompressionError.code
    for i in (0, 3):
        check_vs_oracle(bt, i, probs[i], svs[i])


@pytest.mark.parametrize("N,n2,B", [(700, 150, 3), (1100, 250, 2)])
def test_factor_batched_pivoting(N, n2, B):
    # prescribed-spectrum matrices (many 2x2 pivots and interchanges) through
    # mds_factor_batched + mds_solve_batched directly
    mats = [mdsgen.g3_prescribed(N, seed=N + i, n2x2=n2) for i in range(B)]
    ldm = N + (N % 2)
    M = torch.zeros((B, ldm * N), dtype=torch.float64, device="cuda")
    for i, (A, _) in enumerate(mats):
        host = np.zeros((N, ldm))
        host[:, :N] = np.asarray(A).T
        M[i] = torch.from_numpy(host.reshape(-1))
    piv = torch.empty((B, 2 * N), dtype=torch.int32, device="cuda")
    ine = torch.zeros((B, 3), dtype=torch.int64, device="cuda")
    status = torch.zeros(B, dtype=torch.int32, device="cuda")
    fwork = torch.empty(mds.factor_batched_workspace_size(N, B), dtype=torch.uint8, device="cuda")
    swork = torch.empty(mds.solve_batched_workspace_size(N, B), dtype=torch.uint8, device="cuda")
    rng = np.random.default_rng(N)
    bs = rng.standard_normal((B, N))
    rhs = torch.from_numpy(bs).cuda()
    x = torch.empty((B, N), dtype=torch.float64, device="cuda")
    mds.factor_batched(B, N, M, ldm, ldm * N, piv, 2 * N, -1.0, ine, status, fwork)
    mds.solve_batched(None, B, N, M, ldm, ldm * N, piv, 2 * N, rhs, N, None, 0, None, 0, None, 0, x, N, None, 0,
                      -1.0, fwork, status, swork)
    torch.cuda.synchronize()
    assert (status.cpu().numpy() == 0).all()
    for i, (A, ine_exp) in enumerate(mats):
        LD, ipiv, _ = oracle.bk_factor(A)
        tol = oracle.default_tol(A)
        assert tuple(ine[i].tolist()) == oracle.inertia(LD, ipiv, tol) == tuple(ine_exp)
        x_or = oracle.bk_solve(LD, ipiv, bs[i], tol)
        assert rel_inf(x[i].cpu().numpy(), x_or) <= 1e-8


@pytest.mark.slow
def test_batched_c4_full_size_vs_oracle():
    # C4 scenarios at full size (N = 2048, n_s = 131072, bus-local pattern) through the batched path
    base = mdsgen.scopf_base()
    ids = [0, 101, 255]
    probs, svs = scen(base, ids, seed=4000)
    bt = mds.BatchedKKTStep(probs, svs=svs)
    g = bt.capture()
    g.replay()
    for i in range(len(ids)):
        check_vs_oracle(bt, i, probs[i], svs[i])


@pytest.fixture
def ozaki_variant():
    mds.set_variant("default")
    mds.set_variant("ozaki", 1)
    yield
    mds.set_variant("default")


@pytest.mark.parametrize("N,n2,B", [(700, 150, 3), (1100, 250, 2)])
def test_factor_batched_pivoting_ozaki(N, n2, B, ozaki_variant):
    # the emulated-FP64 (INT8 tensor-core, Ozaki splitting) trailing update, same parity bars
    test_factor_batched_pivoting(N, n2, B)


def test_batched_step_vs_oracle_ozaki(ozaki_variant):
    test_batched_step_vs_oracle((6000, 100, 40, 60), 4)
