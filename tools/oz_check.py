"""Emulated-FP64 (Ozaki) trailing update: parity vs the oracle and timing A/B (GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import mdsgen, oracle
import paper_2605_13736_b200 as mds
from tests.helpers import rel_inf

def dense_batched(mats, ozaki):
    B = len(mats); N = mats[0][0].shape[0]; ldm = N + (N % 2)
    mds.set_variant("default")
    if ozaki: mds.set_variant("ozaki", 1)
    M = torch.zeros((B, ldm * N), dtype=torch.float64, device="cuda")
    for i, (A, _) in enumerate(mats):
        h = np.zeros((N, ldm)); h[:, :N] = np.asarray(A).T; M[i] = torch.from_numpy(h.reshape(-1))
    piv = torch.empty((B, 2 * N), dtype=torch.int32, device="cuda")
    ine = torch.zeros((B, 3), dtype=torch.int64, device="cuda")
    st = torch.zeros(B, dtype=torch.int32, device="cuda")
    fw = torch.empty(mds.factor_batched_workspace_size(N, B), dtype=torch.uint8, device="cuda")
    sw = torch.empty(mds.solve_batched_workspace_size(N, B), dtype=torch.uint8, device="cuda")
    bs = np.random.default_rng(N).standard_normal((B, N)); rhs = torch.from_numpy(bs).cuda()
    x = torch.empty((B, N), dtype=torch.float64, device="cuda")
    mds.factor_batched(B, N, M, ldm, ldm * N, piv, 2 * N, -1.0, ine, st, fw)
    mds.solve_batched(None, B, N, M, ldm, ldm * N, piv, 2 * N, rhs, N, None, 0, None, 0, None, 0, x, N, None, 0, -1.0, fw, st, sw)
    torch.cuda.synchronize()
    return ine.cpu().numpy(), x.cpu().numpy(), st.cpu().numpy(), bs

for N, n2 in ((300, 60), (700, 150), (1100, 250)):
    mats = [mdsgen.g3_prescribed(N, seed=N + i, n2x2=n2) for i in range(3)]
    for oz in (0, 1):
        ine, x, st, bs = dense_batched(mats, oz)
        errs = []
        for i, (A, e) in enumerate(mats):
            LD, ipiv, _ = oracle.bk_factor(A); tol = oracle.default_tol(A)
            xo = oracle.bk_solve(LD, ipiv, bs[i], tol)
            As = np.tril(A) + np.tril(A, -1).T
            res = np.abs(As @ x[i] - bs[i]).max() / np.abs(bs[i]).max()
            errs.append((tuple(ine[i]) == tuple(e), rel_inf(x[i], xo), res))
        print(f"G3 N={N} ozaki={oz} status={st.tolist()} ", [(a, f"{b:.1e}", f"{c:.1e}") for a, b, c in errs])
# SCOPF-like batched steps vs oracle
base = mdsgen.scopf_base(seed=7, n_s=20000, n_d=300, m_E=100, m_I=200)
probs = [mdsgen.scopf_scenario(base, s, seed=7) for s in range(3)]
mds.set_variant("default"); mds.set_variant("ozaki", 1)
bt = mds.BatchedKKTStep(probs)
bt.run()
for i, p in enumerate(probs):
    out = bt.results(i); ref = oracle.newton_step(p)
    print("scopf", i, out["inertia"] == ref["inertia"], f"{rel_inf(out['dxy'], ref['dxy']):.2e}", out["status"])
mds.set_variant("default")
# timing: C4 batched 256 scenarios update class, DMMA vs Ozaki
if "--time" in sys.argv:
    base = mdsgen.scopf_base()
    B = int(os.environ.get("OZB", "256"))
    bt = mds.BatchedKKTStep((B, lambda i: (mdsgen.scopf_scenario(base, i), None)))
    for oz in (0, 1, 0, 1):
        mds.set_variant("default")
        if oz: mds.set_variant("ozaki", 1)
        bt.run(); torch.cuda.synchronize()
        mds.profile_begin(); bt.run(); prof = mds.profile_end()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); bt.run(); e1.record(); torch.cuda.synchronize()
        ok = all(bt.results(i)["inertia"] == (1024, 0, 1024) for i in range(0, B, max(1, B // 8)))
        print(f"C4 B={B} ozaki={oz}: step {e0.elapsed_time(e1):.2f} ms, update {prof['update'][0]:.2f} ms ({prof['update'][1]} launches), inertia ok {ok}")
