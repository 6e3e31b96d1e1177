"""One small hot-path invocation for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck), run eagerly (no CUDA graph) through the C-ABI.

usage: python tools/sanitize_case.py {c1|c2|g3_700|g4_300|batched|ipm|pipeline}
Exit 0 iff the case ran and matched the oracle's inertia (the sanitizer's own
report decides the rest)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import mdsgen  # noqa: E402
import paper_2605_13736_b200 as mds  # noqa: E402


def dense_case(A):
    N = A.shape[0]
    ldm = N + (N % 2)
    host = np.zeros((N, ldm))
    host[:, :N] = np.asarray(A).T
    M = torch.as_tensor(host.reshape(-1), device="cuda").contiguous()
    piv = torch.empty(2 * N, dtype=torch.int32, device="cuda")
    ine_d = torch.zeros(3, dtype=torch.int64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    fwork = torch.empty(mds.factor_workspace_size(N), dtype=torch.uint8, device="cuda")
    swork = torch.empty(mds.solve_workspace_size(N), dtype=torch.uint8, device="cuda")
    ine = mds.factor(N, M, ldm, piv, -1.0, ine_d, status, fwork, sync=True)
    b = torch.ones(N, dtype=torch.float64, device="cuda")
    x = torch.empty(N, dtype=torch.float64, device="cuda")
    mds.solve(None, N, M, ldm, piv, b, None, None, None, x, None, -1.0, fwork, status, swork)
    torch.cuda.synchronize()
    return tuple(ine), int(status.item())


def main():
    case = sys.argv[1]
    torch.cuda.set_device(0)
    if case in ("c1", "c2"):
        prob = mdsgen.config_problem(case.upper())
        sv = mdsgen.step_vectors_for(prob, seed=1)
        st = mds.KKTStep(mds.DeviceProblem(prob), sv=sv)
        ine = st.run(sync_inertia=True)
        out = st.results()
        ok = tuple(ine) == tuple(prob.expected_inertia) and out["status"] == 0
        print(case, "inertia", ine, "status", out["status"])
    elif case.startswith("g3_"):
        N = int(case[3:])
        A, expected = mdsgen.g3_prescribed(N, seed=7)
        ine, status = dense_case(A)
        ok = ine == tuple(expected) and status == 0
        print(case, "inertia", ine, "expected", expected, "status", status)
    elif case.startswith("g4_"):
        N = int(case[3:])
        A = mdsgen.g4_random_symmetric(N, seed=3, shrink_diag=True)
        ine, status = dense_case(A)
        ok = status == 0 and sum(ine) == N
        print(case, "inertia", ine, "status", status)
    elif case == "batched":
        base = mdsgen.scopf_base(seed=7, n_s=3000, n_d=60, m_E=30, m_I=40)
        probs = [mdsgen.scopf_scenario(base, s, seed=7) for s in range(3)]
        svs = [mdsgen.step_vectors_for(p, seed=100 + s) for s, p in enumerate(probs)]
        bt = mds.BatchedKKTStep(probs, svs=svs)
        bt.run()
        outs = [bt.results(i) for i in range(3)]
        ok = all(o["inertia"] == tuple(p.expected_inertia) and o["status"] == 0 for o, p in zip(outs, probs))
        print(case, [o["inertia"] for o in outs], [o["status"] for o in outs])
    elif case == "ipm":
        # small convex QP, eager: K0 products (mds_kkt_residual tiles), the IPM vector kernels,
        # inertia correction, the hot path per Newton iteration
        from paper_2605_13736_b200.ipm import IPMSolver
        qp = mdsgen.qp_problem(2000, 40, 15, 20, seed=5)
        res = IPMSolver(qp, use_graph=False).solve()
        ok = res["status"] == "Optimal"
        print(case, res["status"], res["iterations"], res["e0"])
    elif case == "pipeline":
        prob = mdsgen.config_problem("C1")
        sv = mdsgen.step_vectors_for(prob, seed=1)
        pipe = mds.HostPipeline(prob, sv=sv, use_graph=False)
        host, hout = pipe.pinned_inputs(), pipe.pinned_outputs()
        pipe.run(3, host, hout)
        torch.cuda.synchronize()
        ok = tuple(int(v) for v in hout[1]) == tuple(prob.expected_inertia)
        print(case, tuple(int(v) for v in hout[1]))
    else:
        raise SystemExit(f"unknown case {case}")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
