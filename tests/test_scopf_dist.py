"""SCOPF scenario batching -- the multi-process logic on
CPU with the gloo backend (world_size 2): round-robin partition, the per-step
global stopping test (MAX/SUM all-reduce) and the final all-gather give the
same answers as a single process.  The per-scenario KKT work here is the CPU
oracle (the CUDA path is covered by tests/test_gpu_scopf.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import mdsgen
import oracle
from paper_2605_13736_b200 import scopf

N_SCEN = 7


def scenario_records(ids, base):
    recs = []
    for s in ids:
        p = mdsgen.scopf_scenario(base, s, seed=11)
        out = oracle.newton_step(p)
        sv = mdsgen.step_vectors_for(p, seed=100 + s)
        dx = np.concatenate([out["dx_s"], out["dxy"][:p.n_d]])
        _, v, _ = oracle.step_vectors(sv.x, dx, sv.lo, sv.up, sv.zl, sv.zu, sv.dzl, sv.dzu, sv.tau, sv.mu)
        recs.append([s, *out["inertia"], v["alpha_p"], v["alpha_d"], oracle.norm_inf(p.r), v["compl_inf"]])
    return torch.tensor(recs, dtype=torch.float64).reshape(-1, scopf.REC)


def small_base():
    return mdsgen.scopf_base(seed=11, n_s=300, n_d=12, m_E=6, m_I=6, pattern="uniform")


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    base = small_base()
    ids = scopf.partition(N_SCEN, world, rank)
    rec = scenario_records(ids, base)
    mx, sm = scopf.stats_vector(rec, (base.n_d, 0, base.m))
    stats = scopf.global_stats(mx, sm)
    allr = scopf.gather_records(rec, N_SCEN)
    if rank == 0:
        q.put((stats, allr))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partition_round_robin():
    parts = [scopf.partition(10, 4, r) for r in range(4)]
    assert sorted(sum(parts, [])) == list(range(10))
    assert parts[1] == [1, 5, 9]


def test_two_rank_gloo_matches_single_process():
    base = small_base()
    rec1 = scenario_records(range(N_SCEN), base)
    mx, sm = scopf.stats_vector(rec1, (base.n_d, 0, base.m))
    stats1 = scopf.global_stats(mx, sm)
    all1 = scopf.gather_records(rec1, N_SCEN)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    stats2, all2 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    np.testing.assert_array_equal(all2, all1)          # bitwise: same per-scenario work
    assert stats2 == stats1
    assert stats1["n_scenarios"] == N_SCEN and stats1["n_bad_inertia"] == 0
    assert not stats1["any_bad_inertia"]


def test_stats_flags_bad_inertia():
    rec = torch.tensor([[0, 12, 0, 12, 0.5, 0.6, 1.0, 2.0], [1, 11, 0, 13, 0.4, 0.7, 3.0, 1.0]],
                       dtype=torch.float64)
    mx, sm = scopf.stats_vector(rec, (12, 0, 12))
    st = scopf.global_stats(mx, sm)
    assert st["n_bad_inertia"] == 1 and st["any_bad_inertia"]
    assert st["min_alpha_p"] == 0.4 and st["min_alpha_d"] == 0.6 and st["max_res_inf"] == 3.0
