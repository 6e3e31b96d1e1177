"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle on the same
seeded inputs.  Bars (BASELINE.json north_star):
  inertia bit-exact; ||x_gpu - x_or||_inf/||x_or||_inf <= 1e-8; relative
  residual ||M x - b||_inf/||b||_inf <= 1e-10 on well-conditioned inputs;
  condensation M within 1e-13 (relative to ||M||_max), w bit-exact;
  step vectors: alpha/compl_inf/sigma bit-exact, sums 1e-12."""
import numpy as np
import pytest

import mdsgen
import oracle
from tests.helpers import rel_inf, sym_from_lower

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2605_13736_b200 as mds  # noqa: E402

X_TOL = 1e-8
RES_TOL = 1e-10


def run_step(prob, sv=None, zero_tol=-1.0):
    dp = mds.DeviceProblem(prob)
    st = mds.KKTStep(dp, sv=sv, zero_tol=zero_tol)
    st.run(sync_inertia=True)
    torch.cuda.synchronize()
    return st, st.results()


def upload_dense(A):
    """Run only the factor+solve on an arbitrary symmetric matrix (lower used)."""
    N = A.shape[0]
    ldm = N + (N % 2)
    M = torch.zeros(ldm * N, dtype=torch.float64, device="cuda")
    host = np.zeros((N, ldm))
    host[:, :N] = np.asarray(A).T      # row j of host = column j of A
    M.copy_(torch.from_numpy(host.reshape(-1)))
    return M, ldm


def factor_solve_dense(A, b, zero_tol=-1.0):
    N = A.shape[0]
    M, ldm = upload_dense(A)
    piv = torch.empty(2 * N, dtype=torch.int32, device="cuda")
    ine_d = torch.zeros(3, dtype=torch.int64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    fwork = torch.empty(mds.factor_workspace_size(N), dtype=torch.uint8, device="cuda")
    swork = torch.empty(mds.solve_workspace_size(N), dtype=torch.uint8, device="cuda")
    ine = mds.factor(N, M, ldm, piv, zero_tol, ine_d, status, fwork, sync=True)
    rhs = torch.as_tensor(b, dtype=torch.float64, device="cuda").contiguous()
    x = torch.empty(N, dtype=torch.float64, device="cuda")
    mds.solve(None, N, M, ldm, piv, rhs, None, None, None, x, None, zero_tol, fwork, status, swork)
    torch.cuda.synchronize()
    return ine, x.cpu().numpy(), int(status.item()), piv.cpu().numpy()


def check_x(A, b, x, x_or):
    As = sym_from_lower(A)
    res = np.abs(As @ x - b).max() / np.abs(b).max()
    assert res <= RES_TOL, res
    assert rel_inf(x, x_or) <= X_TOL, rel_inf(x, x_or)


# ---------------------------------------------------------------- condensation
@pytest.mark.parametrize("shape,pattern,dw,dc", [
    ((400, 20, 10, 10), "uniform", 0.0, 0.0),          # C1
    ((3000, 70, 33, 40), "local", 0.01, 1e-8),          # several tiles, ragged
    ((20000, 150, 100, 157), "uniform", 0.0, 0.3),
    ((5000, 0, 60, 70), "local", 0.0, 0.0),             # n_d = 0
    ((4000, 50, 90, 0), "uniform", 0.0, 0.0),           # m_I = 0
    ((4000, 50, 0, 90), "uniform", 0.0, 0.0),           # m_E = 0
    ((0, 40, 10, 10), "uniform", 0.0, 0.0),             # n_s = 0
    ((30000, 130, 200, 170), "local", 1e-3, 0.0),       # bus-local pattern, long runs per destination
])
def test_condense_parity(shape, pattern, dw, dc):
    # w is formed with the elimination's own operations (bit-exact).  M and rhs_c sum the
    # same products in a different (fixed, deterministic) order than the oracle's one
    # sparse variable at a time (readings R7/R8): elementwise within
    # 1e-14 of ||M||_max (a few ulps of the largest entry), and bitwise reproducible.
    prob = mdsgen.g1_quasidefinite(*shape, seed=sum(shape), pattern=pattern, delta_w=dw, delta_c=dc)
    M_or, rhs_or, w_or = oracle.condense(prob)
    dp = mds.DeviceProblem(prob)
    st = mds.KKTStep(dp)
    anorm = torch.full((1,), -1.0, dtype=torch.float64, device="cuda")
    for _ in range(2):   # the workspace (tile queue, norm tickets) must be reusable
        mds.condense(dp.plan, dp.val, dp.h_ss, dp.sigma_s, dp.H_dd, dp.ldh, dp.sigma_d, dp.J_d, dp.ldj, dp.d_h,
                     dp.delta_w, dp.delta_c, dp.r, st.M, st.ldm, st.rhs, st.w, st.status, anorm_out=anorm,
                     work=st.cwork)
    torch.cuda.synchronize()
    M = st.M_host()
    rhs = st.rhs[:prob.N].cpu().numpy()
    if prob.N:
        scale = np.abs(np.tril(M_or)).max()
        assert np.abs(np.tril(M) - np.tril(M_or)).max() <= 1e-14 * scale
        assert np.abs(rhs - rhs_or).max() <= 1e-14 * max(np.abs(rhs_or).max(), 1.0)
    np.testing.assert_array_equal(st.w[:prob.n_s].cpu().numpy(), w_or)
    # bitwise reproducible: a second call gives the same bits
    mds.condense(dp.plan, dp.val, dp.h_ss, dp.sigma_s, dp.H_dd, dp.ldh, dp.sigma_d, dp.J_d, dp.ldj, dp.d_h,
                 dp.delta_w, dp.delta_c, dp.r, st.M, st.ldm, st.rhs, st.w, st.status, anorm_out=anorm,
                 work=st.cwork)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(st.M_host(), M)
    np.testing.assert_array_equal(st.rhs[:prob.N].cpu().numpy(), rhs)
    a_or = oracle.anorm_lower(M_or)
    assert abs(float(anorm.item()) - a_or) <= 1e-13 * a_or
    assert int(st.status.item()) == 0


def test_condense_anorm_deterministic_and_nonfinite():
    prob = mdsgen.g1_quasidefinite(20000, 150, 100, 157, seed=4)
    dp = mds.DeviceProblem(prob)
    st = mds.KKTStep(dp)
    vals = []
    for _ in range(3):
        st.factor_phase(sync_inertia=True)
        vals.append(float(st.anorm.item()))
    assert vals[0] == vals[1] == vals[2]
    # a NaN in the inputs -> anorm_out NaN -> mds_factor reports NONFINITE and factors
    # nothing; the solve issued anyway (as a captured graph would), on a FRESH step whose
    # piv was never written, stays in bounds (identity permutation left by the abort)
    dp.H_dd[5] = float("nan")
    st2 = mds.KKTStep(dp, sv=mdsgen.step_vectors_for(prob, seed=1))
    st2.piv.fill_(1 << 28)
    st2.run()
    torch.cuda.synchronize()
    assert np.isnan(float(st2.anorm.item()))
    assert int(st2.status.item()) == mds.NumericError.code


def test_condense_nonpositive_status():
    prob = mdsgen.g1_quasidefinite(500, 10, 5, 5, seed=2)
    prob.h_ss = prob.h_ss.copy()
    prob.h_ss[7] = -10.0
    dp = mds.DeviceProblem(prob)
    st = mds.KKTStep(dp)
    mds.condense(dp.plan, dp.val, dp.h_ss, dp.sigma_s, dp.H_dd, dp.ldh, dp.sigma_d, dp.J_d, dp.ldj, dp.d_h,
                 dp.delta_w, dp.delta_c, dp.r, st.M, st.ldm, st.rhs, st.w, st.status)
    torch.cuda.synchronize()
    assert int(st.status.item()) == mds.CompressionError.code


def test_plan_rejects_bad_pattern():
    prob = mdsgen.g1_quasidefinite(50, 4, 3, 3, seed=1)
    ci = prob.colidx.copy()
    k = int(np.argmax(np.diff(prob.rowptr) >= 2))
    p = prob.rowptr[k]
    ci[p], ci[p + 1] = ci[p + 1], ci[p]
    with pytest.raises(mds.MalformedMatrixError):
        mds.Plan(prob.n_s, prob.n_d, prob.m_E, prob.m_I, prob.rowptr, ci)


# ---------------------------------------------------------------- factor + solve
@pytest.mark.parametrize("shape", [(400, 20, 10, 10), (2000, 64, 40, 26), (6000, 200, 77, 56),
                                   (30000, 300, 200, 223)])
def test_full_step_parity_quasidefinite(shape):
    prob = mdsgen.g1_quasidefinite(*shape, seed=11 + shape[1])
    sv = mdsgen.step_vectors_for(prob, seed=5)
    st, out = run_step(prob, sv=sv)
    ref = oracle.newton_step(prob)
    assert out["status"] == 0
    assert out["inertia"] == ref["inertia"] == prob.expected_inertia
    check_x(ref["M"], ref["rhs_c"], out["dxy"], ref["dxy"])
    assert rel_inf(out["dx_s"], ref["dx_s"]) <= X_TOL
    # step vectors on the oracle's own direction vs the GPU's: compare to oracle on the GPU direction
    dx = np.concatenate([out["dx_s"], out["dxy"][:prob.n_d]])
    s, v, sig = oracle.step_vectors(sv.x, dx, sv.lo, sv.up, sv.zl, sv.zu, sv.dzl, sv.dzu, sv.tau, sv.mu)
    assert out["vec"]["alpha_p"] == v["alpha_p"]
    assert out["vec"]["alpha_d"] == v["alpha_d"]
    assert out["vec"]["compl_inf"] == v["compl_inf"]
    assert abs(out["vec"]["compl_sum"] - v["compl_sum"]) <= 1e-12 * abs(v["compl_sum"])
    assert out["vec"]["n_compl"] == v["n_compl"] and out["vec"]["first_bad"] == v["first_bad"] == -1
    assert out["vec"]["res_inf"] == oracle.norm_inf(prob.r)
    np.testing.assert_array_equal(out["sigma"], sig)


def test_indefinite_inertia_parity():
    prob = mdsgen.g2_indefinite(3000, 150, 60, 70, seed=5, p_neg=17)
    st, out = run_step(prob)
    ref = oracle.newton_step(prob)
    assert out["inertia"] == ref["inertia"] == prob.expected_inertia
    check_x(ref["M"], ref["rhs_c"], out["dxy"], ref["dxy"])


@pytest.mark.parametrize("N,n2", [(70, 10), (200, 40), (333, 60), (700, 150)])
def test_prescribed_spectrum_pivoting(N, n2):
    # 2x2 pivots and interchanges across panel boundaries (slow path)
    A, ine = mdsgen.g3_prescribed(N, seed=N + 1, n2x2=n2)
    b = np.random.default_rng(N).standard_normal(N)
    LD, ipiv, _ = oracle.bk_factor(A)
    tol = oracle.default_tol(A)
    x_or = oracle.bk_solve(LD, ipiv, b, tol)
    g_ine, x, status, piv = factor_solve_dense(A, b)
    assert status == 0
    assert g_ine == oracle.inertia(LD, ipiv, tol) == ine
    check_x(A, b, x, x_or)


@pytest.mark.parametrize("N", [5, 63, 64, 65, 130, 257])
def test_random_symmetric_shrunk_diag(N):
    A = mdsgen.g4_random_symmetric(N, 3 * N, shrink_diag=True)
    b = np.random.default_rng(N).standard_normal(N)
    LD, ipiv, _ = oracle.bk_factor(A)
    tol = oracle.default_tol(A)
    x_or = oracle.bk_solve(LD, ipiv, b, tol)
    g_ine, x, status, piv = factor_solve_dense(A, b)
    assert g_ine == oracle.inertia(LD, ipiv, tol)
    As = sym_from_lower(A)
    # random symmetric matrices can be ill-conditioned: backward-error gate (R9)
    res = np.abs(As @ x - b).max() / (np.abs(As).sum(1).max() * np.abs(x).max() + np.abs(b).max())
    assert res <= 100 * N * np.finfo(float).eps
    cond = np.linalg.cond(As)
    assert rel_inf(x, x_or) <= max(X_TOL, 100 * N * np.finfo(float).eps * cond)


def test_singular_zero_pivot():
    prob = mdsgen.g5_singular(3000, 40, 30, 30, seed=4)
    st, out = run_step(prob)
    assert out["inertia"] == prob.expected_inertia
    assert out["status"] == mds.SingularError.code


def test_identity_and_small_examples():
    for A, ine in [(np.eye(3), (3, 0, 0)), (np.diag([-1.0, -2.0]), (0, 0, 2)),
                   (np.array([[0.0, 1.0], [1.0, 0.0]]), (1, 0, 1))]:
        b = np.arange(1, A.shape[0] + 1, dtype=float)
        g_ine, x, status, _ = factor_solve_dense(A, b)
        assert g_ine == ine
        np.testing.assert_allclose(sym_from_lower(A) @ x, b, rtol=0, atol=1e-15)


# ---------------------------------------------------------------- zero-pivot tolerance (reading R4)
def _dense_factor(A):
    N = A.shape[0]
    M, ldm = upload_dense(A)
    piv = torch.empty(2 * N, dtype=torch.int32, device="cuda")
    ine_d = torch.zeros(3, dtype=torch.int64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    fwork = torch.empty(mds.factor_workspace_size(N), dtype=torch.uint8, device="cuda")
    ine = mds.factor(N, M, ldm, piv, -1.0, ine_d, status, fwork, sync=True)
    return ine, fwork, int(status.item())


@pytest.mark.parametrize("kind", ["G1", "G3", "G4"])
def test_factor_tol_matches_oracle(kind):
    # the one threshold that decides "zero" in the inertia: tol = N eps ||M||_inf
    if kind == "G1":
        prob = mdsgen.g1_quasidefinite(20000, 150, 100, 157, seed=21)
        A = oracle.condense(prob)[0]
        st = mds.KKTStep(mds.DeviceProblem(prob))
        st.factor_phase(sync_inertia=True)            # norm fused into the condensation
        a_c, t_c = mds.factor_tol(st.fwork)
        assert abs(t_c - oracle.default_tol(A)) <= 1e-13 * oracle.default_tol(A)
    elif kind == "G3":
        A, _ = mdsgen.g3_prescribed(1300, seed=5, n2x2=200)
    else:
        A = mdsgen.g4_random_symmetric(300, seed=9)
    _, fwork, status = _dense_factor(A)                # stand-alone scan inside mds_factor
    a_g, t_g = mds.factor_tol(fwork)
    a_or, t_or = oracle.anorm_lower(A), oracle.default_tol(A)
    assert status == 0
    assert abs(a_g - a_or) <= 1e-13 * a_or and abs(t_g - t_or) <= 1e-13 * t_or


@pytest.mark.parametrize("N,seed", [(300, 1), (1000, 2), (2111, 3)])
def test_pivots_at_the_tolerance(N, seed):
    # G3 plus decoupled 1x1 pivots placed at +-0.5, 0.9, 1.1, 2 and 3 times tol (and 0):
    # their values never change during the elimination (their rows are exactly zero off the
    # diagonal), so whether each counts as zero is decided by the tolerance alone.
    # Expected inertia: closed form, and the oracle's.
    n0 = N - 9
    A0, ine0 = mdsgen.g3_prescribed(n0, seed=seed, n2x2=n0 // 6)
    tol = N * np.finfo(float).eps * oracle.anorm_lower(A0)
    small = np.array([0.5, -0.5, 0.9, -0.9, 0.0, 1.1, -1.1, 2.0, 3.0]) * tol
    B = np.zeros((N, N))
    B[:n0, :n0] = A0
    B[np.arange(n0, N), np.arange(n0, N)] = small
    p = np.random.default_rng(seed).permutation(N)
    B = np.asfortranarray(B[np.ix_(p, p)])
    expected = (ine0[0] + 3, 5, ine0[2] + 1)
    LD, ipiv, _ = oracle.bk_factor(B)
    t_or = oracle.default_tol(B)
    assert oracle.inertia(LD, ipiv, t_or) == expected
    ine, fwork, status = _dense_factor(B)
    assert ine == expected
    assert abs(mds.factor_tol(fwork)[1] - t_or) <= 1e-13 * t_or


def test_nonfinite_input():
    A = mdsgen.g4_random_symmetric(100, 1)
    A[50, 3] = np.inf
    N = 100
    M, ldm = upload_dense(A)
    piv = torch.empty(2 * N, dtype=torch.int32, device="cuda")
    ine_d = torch.zeros(3, dtype=torch.int64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    fwork = torch.empty(mds.factor_workspace_size(N), dtype=torch.uint8, device="cuda")
    mds.factor(N, M, ldm, piv, -1.0, ine_d, status, fwork, sync=True)
    assert int(status.item()) == mds.NumericError.code


# ---------------------------------------------------------------- step vectors
@pytest.mark.parametrize("n", [1, 2, 31, 1000, 100001])
def test_step_vectors_parity(n):
    sv = mdsgen.step_vectors(n, seed=n)
    d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda").contiguous()
    out = torch.zeros(16, dtype=torch.float64, device="cuda")
    sig = torch.empty(n, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    work = torch.zeros(mds.step_vectors_workspace_size(n), dtype=torch.uint8, device="cuda")
    res = d(np.random.default_rng(1).standard_normal(n + 3))
    for _ in range(2):   # workspace must be reusable
        mds.step_vectors(n, d(sv.x), d(sv.dx), d(sv.lo), d(sv.up), d(sv.zl), d(sv.zu), d(sv.dzl), d(sv.dzu),
                         sv.tau, sv.mu, out, sig, status, work, res=(res,))
    torch.cuda.synchronize()
    s, v, sg = oracle.step_vectors(sv.x, sv.dx, sv.lo, sv.up, sv.zl, sv.zu, sv.dzl, sv.dzu, sv.tau, sv.mu)
    o = out.cpu().numpy()
    assert o[0] == v["alpha_p"] and o[1] == v["alpha_d"] and o[2] == v["compl_inf"]
    assert abs(o[3] - v["compl_sum"]) <= 1e-12 * max(abs(v["compl_sum"]), 1e-300)
    assert int(o[4]) == v["n_compl"] and int(o[5]) == v["first_bad"] == -1
    assert o[6] == np.abs(res.cpu().numpy()).max()
    np.testing.assert_array_equal(sig.cpu().numpy(), sg)
    assert int(status.item()) == 0


def test_step_vectors_not_interior():
    sv = mdsgen.step_vectors(5000, seed=3)
    x = sv.x.copy()
    fin = np.where(np.abs(sv.lo) < 1e20)[0]
    x[fin[10]] = sv.lo[fin[10]] - 1.0
    d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda").contiguous()
    out = torch.zeros(16, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    work = torch.zeros(mds.step_vectors_workspace_size(5000), dtype=torch.uint8, device="cuda")
    mds.step_vectors(5000, d(x), d(sv.dx), d(sv.lo), d(sv.up), d(sv.zl), d(sv.zu), d(sv.dzl), d(sv.dzu),
                     sv.tau, sv.mu, out, None, status, work)
    torch.cuda.synchronize()
    s, v, _ = oracle.step_vectors(x, sv.dx, sv.lo, sv.up, sv.zl, sv.zu, sv.dzl, sv.dzu, sv.tau, sv.mu)
    assert int(out[5].item()) == v["first_bad"] == fin[10]
    assert int(status.item()) == mds.NotInteriorError.code


# ---------------------------------------------------------------- graph capture
def test_graph_replay_matches_eager():
    prob = mdsgen.g1_quasidefinite(5000, 100, 50, 50, seed=8)
    sv = mdsgen.step_vectors_for(prob, seed=2)
    dp = mds.DeviceProblem(prob)
    st = mds.KKTStep(dp, sv=sv)
    st.run()
    eager = st.results()
    g = st.capture()
    g.replay()
    rep = st.results()
    assert rep["inertia"] == eager["inertia"]
    np.testing.assert_array_equal(rep["dxy"], eager["dxy"])
    np.testing.assert_array_equal(rep["dx_s"], eager["dx_s"])


# ---------------------------------------------------------------- degenerate sizes
@pytest.mark.parametrize("A,ine", [
    (np.array([[2.5]]), (1, 0, 0)), (np.array([[-3.0]]), (0, 0, 1)),
    (np.array([[0.0, 1.0], [1.0, 0.0]]), (1, 0, 1)),                      # one 2x2 pivot
    (np.array([[1e-3, 2.0, 0.0], [2.0, 1e-3, 1.0], [0.0, 1.0, -4.0]]), None),
])
def test_tiny_dense(A, ine):
    b = np.arange(1.0, A.shape[0] + 1.0)
    LD, ipiv, _ = oracle.bk_factor(np.asfortranarray(np.tril(A)))
    tol = oracle.default_tol(np.tril(A))
    exp = oracle.inertia(LD, ipiv, tol)
    if ine is not None:
        assert exp == ine
    g_ine, x, status, _ = factor_solve_dense(np.tril(A), b)
    assert status == 0 and g_ine == exp
    assert np.abs(A @ x - b).max() <= 1e-12 * np.abs(b).max() * max(1.0, np.abs(A).max())


def test_singular_1x1():
    g_ine, x, status, _ = factor_solve_dense(np.array([[0.0]]), np.array([1.0]))
    assert g_ine == (0, 1, 0) and status == mds.SingularError.code


@pytest.mark.parametrize("shape", [(0, 30, 10, 12), (3000, 64, 64, 0), (2500, 0, 40, 24), (777, 63, 1, 1),
                                   (4000, 50, 0, 90)])
def test_full_step_edge_shapes(shape):
    # no sparse block, no inequalities, no dense variables, N = 65 (one full panel + 1)
    prob = mdsgen.g1_quasidefinite(*shape, seed=3 + sum(shape))
    st, out = run_step(prob)
    ref = oracle.newton_step(prob)
    assert out["status"] == 0
    assert out["inertia"] == ref["inertia"] == prob.expected_inertia
    check_x(ref["M"], ref["rhs_c"], out["dxy"], ref["dxy"])
    if prob.n_s:
        assert rel_inf(out["dx_s"], ref["dx_s"]) <= X_TOL
