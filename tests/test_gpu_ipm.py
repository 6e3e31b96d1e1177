"""The device interior-point loop (paper_2605_13736_b200.ipm.IPMSolver: the hot
path + the IPM vector kernels through the C-ABI) against the oracle's IPM
(oracle/ipm.py) on the same seeded convex QPs: both Optimal, the same barrier
parameter sequence and iteration count, the same solution within the stopping
tolerance's reach, and the KKT conditions at the device solution on a dense
assembly (tests/helpers.dense_qp_parts)."""
import numpy as np
import pytest

import mdsgen
from oracle import ipm as oipm
from tests.helpers import dense_qp_parts

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2605_13736_b200.ipm import IPMSolver  # noqa: E402

INF = 1e20


@pytest.mark.parametrize("shape,seed,pattern", [((400, 20, 10, 10), 1, "uniform"), ((3000, 60, 30, 40), 2, "local"),
                                                ((5000, 80, 0, 50), 3, "uniform"), ((20000, 200, 100, 100), 4, "local"),
                                                ((2000, 30, 25, 0), 9, "uniform")])
def test_device_ipm_matches_oracle(shape, seed, pattern):
    qp = mdsgen.qp_problem(*shape, seed=seed, pattern=pattern)
    ref = oipm.solve(qp)
    sol = IPMSolver(qp)
    res = sol.solve()
    assert ref["status"] == res["status"] == "Optimal"
    assert res["e0"] <= 1e-8
    mus_ref = [h["mu"] for h in ref["history"]]
    mus = [h["mu"] for h in res["history"]]
    assert res["iterations"] == ref["iterations"], (res["iterations"], ref["iterations"])
    np.testing.assert_allclose(mus, mus_ref, rtol=1e-12)
    out = sol.solution()
    assert np.abs(out["x"] - ref["x"]).max() <= 1e-6 * max(1.0, np.abs(ref["x"]).max())
    H, J = dense_qp_parts(qp)
    m_E = qp.base.m_E
    assert np.abs(H @ out["x"] + qp.c + J.T @ out["y"] - out["zl"] + out["zu"]).max() <= 1e-7
    assert np.abs(J[:m_E] @ out["x"] - qp.g_E).max(initial=0.0) <= 1e-7
    assert np.abs(J[m_E:] @ out["x"] - out["s"]).max(initial=0.0) <= 1e-7
    assert all(h["inertia"] == (qp.base.n_d, 0, qp.base.m) for h in res["history"])


@pytest.mark.parametrize("k", [2, 10, 100, 1000])
def test_device_ipm_nlpmds_ex4(k):
    # the paper's mini-app problem: compressed size 2k+3, optimum x = 1/2 (closed form)
    qp = mdsgen.synthetic_problem(k)
    ref = oipm.solve(qp)
    sol = IPMSolver(qp)
    res = sol.solve()
    assert res["status"] == ref["status"] == "Optimal"
    assert res["iterations"] == ref["iterations"]
    assert np.abs(sol.solution()["x"] - 0.5).max() <= 1e-7
