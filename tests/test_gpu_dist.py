"""Distributed LDL^T of one system (paper_2605_13736_b200.dist, SURVEY §8(f)
NEXT-4) through the CUDA path against the CPU oracle's Bunch-Kaufman
(oracle.bk_factor / inertia / bk_solve): inertia exact, x within 1e-8.  World
size 1 in process, and 2 ranks as two processes sharing the one GPU (gloo; the
NCCL path is the same code with device tensors).  Cases: a quasi-definite
condensed M (every panel accepted: the distributed phase only), a pivot-heavy
prescribed-spectrum matrix (the exact phase from the first panel), and a matrix
whose speculative panels fail part-way (both phases)."""
import os
import socket

import numpy as np
import pytest

import mdsgen
import oracle
from tests.helpers import rel_inf

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2605_13736_b200 import dist as pdist  # noqa: E402


def quasi_definite(N_target=1000, seed=41):
    p = mdsgen.g1_quasidefinite(n_s=4000, n_d=N_target // 2, m_E=N_target // 4, m_I=N_target - N_target // 2 - N_target // 4,
                                seed=seed)
    return oracle.newton_step(p)["M"]


def mid_failure(seed=43):
    # quasi-definite, with rows/columns k, k+1 replaced by the 2x2 block [[0, 1], [1, 0]]
    # (plus a coupling below): the panel holding k fails the 1x1 test (Bunch-Kaufman needs a
    # 2x2 pivot there) and the distributed phase ends at it (both phases run)
    M = np.array(quasi_definite(900, seed), copy=True)
    k = 707
    M[k:k + 2, :] = 0.0
    M[:, k:k + 2] = 0.0
    M[k + 1, k] = 1.0
    M[k + 5, k] = 0.3
    M[k + 9, k + 1] = -0.2
    return M


def cases():
    return {"quasi_definite": lambda: quasi_definite(1000, 41),
            "pivot_heavy": lambda: mdsgen.g3_prescribed(700, seed=42, n2x2=150)[0],
            "mid_failure": mid_failure}


def reference(M, b):
    M = np.asarray(M)
    LD, ipiv, _ = oracle.bk_factor(M)
    tol = oracle.default_tol(M)
    return oracle.inertia(LD, ipiv, tol), oracle.bk_solve(LD, ipiv, b, tol)


def run_rank(M, b):
    N = M.shape[0]
    d = pdist.DistLDLT(N)
    d.load_full(M)
    ine = d.factor()
    x = d.solve(torch.from_numpy(b).cuda())
    torch.cuda.synchronize()
    return ine, x.cpu().numpy(), d.pf, d.np


@pytest.mark.parametrize("case", list(cases()))
def test_dist_world1_vs_oracle(case):
    M = np.asarray(cases()[case]())
    b = np.random.default_rng(7).standard_normal(M.shape[0])
    ine, x, pf, npanel = run_rank(M, b)
    ine_ref, x_ref = reference(M, b)
    assert ine == ine_ref
    assert rel_inf(x, x_ref) <= 1e-8, rel_inf(x, x_ref)
    if case == "quasi_definite":
        assert pf == npanel          # never left the distributed phase
    if case == "mid_failure":
        assert 0 < pf < npanel       # both phases


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        M = np.asarray(cases()[case]())
        b = np.random.default_rng(7).standard_normal(M.shape[0])
        ine, x, pf, npanel = run_rank(M, b)
        q.put((rank, ine, x, pf, npanel))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("case", list(cases()))
def test_dist_two_ranks_vs_oracle(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    M = np.asarray(cases()[case]())
    b = np.random.default_rng(7).standard_normal(M.shape[0])
    ine_ref, x_ref = reference(M, b)
    for rank, ine, x, pf, npanel in res:
        assert ine == ine_ref, (rank, ine, ine_ref)
        assert rel_inf(x, x_ref) <= 1e-8, (rank, rel_inf(x, x_ref))
    # the two ranks hold the same solution (replicated by the broadcasts)
    np.testing.assert_array_equal(res[0][2], res[1][2])
