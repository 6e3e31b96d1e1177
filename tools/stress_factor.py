"""Randomised GPU stress of mds_factor + mds_solve on pivot-heavy matrices (not a
unit test: a sweep over sizes, spectra and launch-structure variants, run on the
GPU box).  Each case: inertia must equal the closed form (G3) / the oracle (G4),
and the residual of the original system must be <= 1e-10 (G3) or the
backward-error bound (G4).  Prints one line per case and a summary; exit 1 on
any failure.  usage: python tools/stress_factor.py [n_cases] [seed]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mdsgen  # noqa: E402
import oracle  # noqa: E402
import paper_2605_13736_b200 as mds  # noqa: E402

VARIANTS = [{}, {"tail_rows": 0}, {"tail_rows": 100000000}, {"exact_no_ls": 1},
            {"f2_trsm": 1}, {"no_pdl": 1}, {"CAP": 8}, {"CAP": 37}]


def run(A, b):
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
    rhs = torch.as_tensor(b, device="cuda").contiguous()
    x = torch.empty(N, dtype=torch.float64, device="cuda")
    mds.solve(None, N, M, ldm, piv, rhs, None, None, None, x, None, -1.0, fwork, status, swork)
    torch.cuda.synchronize()
    return tuple(ine), x.cpu().numpy(), int(status.item())


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    fails = 0
    t0 = time.time()
    for case in range(n):
        var = VARIANTS[case % len(VARIANTS)]
        mds.set_variant("default")
        for k, v in var.items():
            if k != "CAP":
                mds.set_variant(k, v)
        mds.set_grid_cap(int(var.get("CAP", "0")))   # concurrent-factorization launch structure
        kind = "G3" if case % 3 else "G4"
        N = int(rng.integers(65, int(os.environ.get("STRESS_NMAX", "3500")) if kind == "G3" else 700))
        b = rng.standard_normal(N)
        if kind == "G3":
            A, ine_exp = mdsgen.g3_prescribed(N, seed=int(rng.integers(1 << 30)), n2x2=int(rng.integers(0, N // 3)))
        else:
            A = mdsgen.g4_random_symmetric(N, int(rng.integers(1 << 30)), shrink_diag=bool(rng.integers(2)))
            LD, ipiv, _ = oracle.bk_factor(A)
            ine_exp = oracle.inertia(LD, ipiv, oracle.default_tol(A))
        ine, x, st = run(A, b)
        As = np.tril(A) + np.tril(A, -1).T
        r = np.abs(As @ x - b).max()
        if kind == "G3":
            ok = st == 0 and ine == tuple(ine_exp) and r / np.abs(b).max() <= 1e-10
            err = r / np.abs(b).max()
        else:
            err = r / (np.abs(As).sum(1).max() * np.abs(x).max() + np.abs(b).max())
            ok = st == 0 and ine == tuple(ine_exp) and err <= 100 * N * np.finfo(float).eps
        fails += 0 if ok else 1
        print(f"{'ok  ' if ok else 'FAIL'} case {case:3d} {kind} N={N:5d} var={var} inertia={ine} exp={tuple(ine_exp)} "
              f"err={err:.2e} status={st}", flush=True)
    print(f"{n - fails}/{n} passed in {time.time() - t0:.0f} s")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
