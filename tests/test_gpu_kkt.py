"""mds_kkt_residual (K2 mat-vec of the full Eq.(5) matrix) against the oracle's
kkt_matvec, and the whole Newton step checked against the ORIGINAL system:
||r - K [dx_s; dx_d; dy]||_inf / ||r||_inf <= 1e-10 at C2 and C3 sizes (the
condensation + BK + solve + recovery chain is exact up to rounding)."""
import numpy as np
import pytest

import mdsgen
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2605_13736_b200 as mds  # noqa: E402


def gpu_residual(dp, x, b=None):
    out = torch.empty_like(x)
    rn = torch.zeros(1, dtype=torch.float64, device="cuda")
    mds.kkt_residual(dp.plan, dp.val, dp.h_ss, dp.sigma_s, dp.H_dd, dp.ldh, dp.sigma_d, dp.J_d, dp.ldj, dp.d_h,
                     dp.delta_w, dp.delta_c, x, b, out, rn)
    torch.cuda.synchronize()
    return out.cpu().numpy(), float(rn.item())


@pytest.mark.parametrize("shape,dw,dc", [((400, 20, 10, 10), 0.0, 0.0), ((3000, 70, 33, 40), 0.01, 1e-8),
                                         ((5000, 0, 60, 70), 0.0, 0.2), ((0, 40, 10, 10), 0.0, 0.0),
                                         ((100000, 512, 256, 256), 0.0, 0.0)])
def test_matvec_parity(shape, dw, dc):
    q = mdsgen.g1_quasidefinite(*shape, seed=sum(shape), delta_w=dw, delta_c=dc)
    dp = mds.DeviceProblem(q)
    n = q.n_s + q.n_d + q.m_E + q.m_I
    x = np.random.default_rng(5).standard_normal(n)
    kx, _ = gpu_residual(dp, torch.as_tensor(x, device="cuda"))
    ref = oracle.kkt_matvec(q, x)
    assert np.abs(kx - ref).max() <= 1e-13 * np.abs(ref).max()
    b = np.random.default_rng(6).standard_normal(n)
    res, rn = gpu_residual(dp, torch.as_tensor(x, device="cuda"), torch.as_tensor(b, device="cuda"))
    assert np.abs(res - (b - ref)).max() <= 1e-13 * np.abs(b - ref).max()
    assert rn == np.abs(res).max()


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_newton_step_solves_original_system(cfg):
    q = mdsgen.config_problem(cfg)
    dp = mds.DeviceProblem(q)
    st = mds.KKTStep(dp)
    g = st.capture()
    g.replay()
    torch.cuda.synchronize()
    st.check_status()
    x = torch.cat([st.dx_s, st.dxy])
    res, rn = gpu_residual(dp, x, dp.r)
    rinf = float(dp.r.abs().max().item())
    assert rn / rinf <= 1e-10, rn / rinf
    # the same residual from the oracle's mat-vec on the GPU's direction
    ref = np.asarray(q.r) - oracle.kkt_matvec(q, x.cpu().numpy())
    assert np.abs(ref).max() / rinf <= 1e-10
