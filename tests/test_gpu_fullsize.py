"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (CUDA-graph replay of the whole step):
  C2 (N=1024, n_s=100k): every output against the oracle.
  C3 (N=8192, n_s=1M): condensed M and rhs_c element by element within 1e-14 of
    their largest entry, w bit-exact, ||M||_inf within 1e-13; inertia against the closed form AND the oracle's BK
    factorization; the solution element by element against the oracle's
    (<= 1e-8) and through the residual of the condensed system (<= 1e-10);
    step vectors against the oracle on the GPU's direction.
  C4 (one full-size SCOPF scenario, N=2048, n_s=131072): every output vs the oracle."""
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


def graph_step(prob, sv):
    st = mds.KKTStep(mds.DeviceProblem(prob), sv=sv)
    g = st.capture()
    g.replay()
    torch.cuda.synchronize()
    return st, st.results()


def sym_matvec_lower(M, x):
    L = np.tril(M)
    return L @ x + np.tril(M, -1).T @ x


def test_c2_full_step_vs_oracle():
    prob = mdsgen.config_problem("C2")
    sv = mdsgen.step_vectors_for(prob, seed=7)
    st, out = graph_step(prob, sv)
    ref = oracle.newton_step(prob)
    assert out["status"] == 0
    assert out["inertia"] == ref["inertia"] == prob.expected_inertia
    assert rel_inf(out["dxy"], ref["dxy"]) <= 1e-8
    assert rel_inf(out["dx_s"], ref["dx_s"]) <= 1e-8
    res = np.abs(sym_matvec_lower(ref["M"], out["dxy"]) - ref["rhs_c"]).max() / np.abs(ref["rhs_c"]).max()
    assert res <= 1e-10


def test_c3_full_size_properties():
    prob = mdsgen.config_problem("C3")
    sv = mdsgen.step_vectors_for(prob, seed=7)
    dp = mds.DeviceProblem(prob)
    st = mds.KKTStep(dp, sv=sv)
    # condensation alone, element by element
    anorm = torch.zeros(1, dtype=torch.float64, device="cuda")
    mds.condense(dp.plan, dp.val, dp.h_ss, dp.sigma_s, dp.H_dd, dp.ldh, dp.sigma_d, dp.J_d, dp.ldj, dp.d_h,
                 dp.delta_w, dp.delta_c, dp.r, st.M, st.ldm, st.rhs, st.w, st.status, anorm_out=anorm,
                 work=st.cwork)
    torch.cuda.synchronize()
    M_or, rhs_or, w_or = oracle.condense(prob)
    Mg = st.M_host()
    assert np.abs(np.tril(Mg) - np.tril(M_or)).max() <= 1e-14 * np.abs(np.tril(M_or)).max()
    np.testing.assert_array_equal(st.w[:prob.n_s].cpu().numpy(), w_or)
    assert rel_inf(st.rhs[:prob.N].cpu().numpy(), rhs_or) <= 1e-14
    a_or = oracle.anorm_lower(M_or)
    assert abs(float(anorm.item()) - a_or) <= 1e-13 * a_or
    del Mg
    # the whole step as bench.py runs it (graph replay)
    g = st.capture()
    g.replay()
    out = st.results()
    assert out["status"] == 0
    assert out["inertia"] == prob.expected_inertia == (4096, 0, 4096)
    res = np.abs(sym_matvec_lower(M_or, out["dxy"]) - rhs_or).max() / np.abs(rhs_or).max()
    assert res <= 1e-10, res
    dy = out["dxy"][prob.n_d:]
    dxs_ref = oracle.recover(prob, w_or, prob.r[:prob.n_s], dy)
    assert rel_inf(out["dx_s"], dxs_ref) <= 1e-12
    # the oracle's own BK factorization + solve at full size (OpenMP, bit-identical to 1 thread)
    ga, gt = mds.factor_tol(st.fwork)
    tol_or = oracle.default_tol(M_or)
    assert abs(gt - tol_or) <= 1e-13 * tol_or
    LD, ipiv, _ = oracle.bk_factor(M_or)
    assert oracle.inertia(LD, ipiv, tol_or) == out["inertia"]
    x_or = oracle.bk_solve(LD, ipiv, rhs_or, tol_or)
    del LD
    assert rel_inf(out["dxy"], x_or) <= 1e-8, rel_inf(out["dxy"], x_or)
    dxs_or = oracle.recover(prob, w_or, prob.r[:prob.n_s], x_or[prob.n_d:])
    assert rel_inf(out["dx_s"], dxs_or) <= 1e-8
    dx = np.concatenate([out["dx_s"], out["dxy"][:prob.n_d]])
    s, v, sig = oracle.step_vectors(sv.x, dx, sv.lo, sv.up, sv.zl, sv.zu, sv.dzl, sv.dzu, sv.tau, sv.mu)
    assert out["vec"]["alpha_p"] == v["alpha_p"] and out["vec"]["alpha_d"] == v["alpha_d"]
    assert out["vec"]["compl_inf"] == v["compl_inf"]
    np.testing.assert_array_equal(out["sigma"], sig)


def test_c4_scenario_full_size_vs_oracle():
    # one SCOPF contingency scenario at the C4 size (N = 2048, n_s = 131072, bus-local pattern)
    base = mdsgen.scopf_base()
    prob = mdsgen.scopf_scenario(base, 37)
    sv = mdsgen.step_vectors_for(prob, seed=37)
    st, out = graph_step(prob, sv)
    ref = oracle.newton_step(prob)
    assert out["status"] == 0
    assert out["inertia"] == ref["inertia"] == prob.expected_inertia
    assert rel_inf(out["rhs_c"], ref["rhs_c"]) <= 1e-14
    np.testing.assert_array_equal(out["w"], ref["w"])
    assert rel_inf(out["dxy"], ref["dxy"]) <= 1e-8
    assert rel_inf(out["dx_s"], ref["dx_s"]) <= 1e-8
    res = np.abs(sym_matvec_lower(ref["M"], out["dxy"]) - ref["rhs_c"]).max() / np.abs(ref["rhs_c"]).max()
    assert res <= 1e-10


@pytest.mark.parametrize("N,n2", [(1500, 300), (2111, 500)])
def test_pivoting_heavy_multi_panel(N, n2):
    # prescribed-spectrum matrices: many 2x2 pivots and interchanges across ~30 panels
    A, ine = mdsgen.g3_prescribed(N, seed=N, n2x2=n2)
    b = np.random.default_rng(N).standard_normal(N)
    LD, ipiv, _ = oracle.bk_factor(A)
    tol = oracle.default_tol(A)
    x_or = oracle.bk_solve(LD, ipiv, b, tol)
    from tests.test_gpu_parity import factor_solve_dense
    g_ine, x, status, _ = factor_solve_dense(A, b)
    assert status == 0
    assert g_ine == oracle.inertia(LD, ipiv, tol) == ine
    As = np.tril(A) + np.tril(A, -1).T
    assert np.abs(As @ x - b).max() / np.abs(b).max() <= 1e-10
    assert rel_inf(x, x_or) <= 1e-8


# The factorization has several launch-structure variants chosen by size or by
# the explicit mds_set_variant API; each must give the same BK answer.  "odd ldm"
# disables the TMA path (16-byte alignment), so the cp.async update kernel
# without look-ahead runs.
@pytest.fixture
def variant_reset():
    yield
    mds.set_variant("default")


@pytest.mark.parametrize("variant", ["tail_always", "tail_never", "no_lookahead", "no_tma", "odd_ldm", "no_pdl",
                                     "static_sched", "upd_main", "inplace", "slow_1cta", "exact_no_ls", "f2_trsm",
                                     "exact_rows_64", "exact_cluster"])
def test_factor_variants_pivoting(variant, variant_reset):
    knobs = {"tail_always": {"tail_rows": 100000000}, "tail_never": {"tail_rows": 0},
             "no_lookahead": {"no_lookahead": 1}, "no_tma": {"no_tma": 1}, "odd_ldm": {},
             "no_pdl": {"no_pdl": 1}, "static_sched": {"static_sched": 1},
             "upd_main": {"upd_main": 1}, "inplace": {"upd_inplace": 1},
             "slow_1cta": {"slow_1cta": 1}, "exact_no_ls": {"exact_no_ls": 1},
             "f2_trsm": {"f2_trsm": 1}, "exact_rows_64": {"exact_rows": 64},
             "exact_cluster": {"exact_cluster": 1}}[variant]
    for k, v in knobs.items():
        mds.set_variant(k, v)
    N, n2 = 1500, 300
    A, ine = mdsgen.g3_prescribed(N, seed=7 * N, n2x2=n2)
    b = np.random.default_rng(N + 1).standard_normal(N)
    LD, ipiv, _ = oracle.bk_factor(A)
    tol = oracle.default_tol(A)
    x_or = oracle.bk_solve(LD, ipiv, b, tol)
    ldm = N + 1 if variant == "odd_ldm" else N
    M = torch.zeros(ldm * N, dtype=torch.float64, device="cuda")
    host = np.zeros((N, ldm))
    host[:, :N] = np.tril(A).T            # row j of host = column j of A (column-major M)
    M.copy_(torch.as_tensor(host.reshape(-1)))
    piv = torch.empty(2 * N, dtype=torch.int32, device="cuda")
    ine_d = torch.zeros(3, dtype=torch.int64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    fwork = torch.empty(mds.factor_workspace_size(N), dtype=torch.uint8, device="cuda")
    swork = torch.empty(mds.solve_workspace_size(N), dtype=torch.uint8, device="cuda")
    g_ine = mds.factor(N, M, ldm, piv, -1.0, ine_d, status, fwork, sync=True)
    rhs = torch.as_tensor(b, dtype=torch.float64, device="cuda").contiguous()
    x = torch.empty(N, dtype=torch.float64, device="cuda")
    mds.solve(None, N, M, ldm, piv, rhs, None, None, None, x, None, -1.0, fwork, status, swork)
    torch.cuda.synchronize()
    x = x.cpu().numpy()
    assert int(status.item()) == 0
    assert g_ine == oracle.inertia(LD, ipiv, tol) == ine
    As = np.tril(A) + np.tril(A, -1).T
    assert np.abs(As @ x - b).max() / np.abs(b).max() <= 1e-10
    assert rel_inf(x, x_or) <= 1e-8


@pytest.mark.parametrize("N,n2", [(8192, 2000), (12289, 100)])
def test_pivoting_heavy_large(N, n2):
    # multi-CTA exact BK panels (k_panel_exact with 32-48 CTAs and grid barriers) on
    # prescribed-spectrum matrices: inertia against the closed form, solve by the residual
    A, ine = mdsgen.g3_prescribed_torch(N, seed=N + 11, n2x2=n2, device="cuda")
    M = A.T.contiguous().reshape(-1)
    piv = torch.empty(2 * N, dtype=torch.int32, device="cuda")
    ine_d = torch.zeros(3, dtype=torch.int64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    fwork = torch.empty(mds.factor_workspace_size(N), dtype=torch.uint8, device="cuda")
    swork = torch.empty(mds.solve_workspace_size(N), dtype=torch.uint8, device="cuda")
    g_ine = mds.factor(N, M, N, piv, -1.0, ine_d, status, fwork, sync=True)
    b = torch.as_tensor(np.random.default_rng(N).standard_normal(N), dtype=torch.float64, device="cuda")
    x = torch.empty(N, dtype=torch.float64, device="cuda")
    mds.solve(None, N, M, N, piv, b, None, None, None, x, None, -1.0, fwork, status, swork)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    assert g_ine == ine
    res = float((A @ x - b).abs().max() / b.abs().max())
    assert res <= 1e-10, res


def test_c5_factor_solve_32768():
    # C5: N = 32768 prescribed-spectrum indefinite matrix (8.6 GB), factor + solve in the
    # launch configuration bench.py --config C5 times; inertia against the closed form,
    # the solve through the residual of the original system (the oracle cannot run at this size)
    N = 32768
    A, ine = mdsgen.g3_prescribed_torch(N, seed=5005, device="cuda")
    M = A.T.contiguous().reshape(-1)          # column-major (A is symmetric; lower used)
    piv = torch.empty(2 * N, dtype=torch.int32, device="cuda")
    ine_d = torch.zeros(3, dtype=torch.int64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    fwork = torch.empty(mds.factor_workspace_size(N), dtype=torch.uint8, device="cuda")
    swork = torch.empty(mds.solve_workspace_size(N), dtype=torch.uint8, device="cuda")
    g_ine = mds.factor(N, M, N, piv, -1.0, ine_d, status, fwork, sync=True)
    b = torch.as_tensor(np.random.default_rng(N).standard_normal(N), dtype=torch.float64, device="cuda")
    x = torch.empty(N, dtype=torch.float64, device="cuda")
    mds.solve(None, N, M, N, piv, b, None, None, None, x, None, -1.0, fwork, status, swork)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    assert g_ine == ine
    res = float((A @ x - b).abs().max() / b.abs().max())
    assert res <= 1e-10, res


@pytest.mark.parametrize("N,n2", [(1500, 300), (2111, 500)])
def test_pivoting_heavy_ozaki_single(N, n2, variant_reset):
    # single-system factorization with the emulated-FP64 update (non-look-ahead launch structure)
    mds.set_variant("no_lookahead", 1)
    mds.set_variant("ozaki", 1)
    test_pivoting_heavy_multi_panel(N, n2)
