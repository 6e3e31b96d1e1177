"""Security-constrained OPF scenario batching (north star:
"Independent contingency KKT systems are batched per GPU across the 8xB200
box, and NCCL over NVLink is used only to gather per-scenario results and the
global stopping test").

One process per GPU.  Rank r owns the scenarios s with s % P == r (round-robin,
so scenarios that converge at different iteration counts stay balanced).  The
local scenarios form ONE `BatchedKKTStep` (all share the pattern plan): a
Newton step for all of them is one CUDA graph of batched launches
(mds_condense_batched / mds_factor_batched / mds_solve_batched /
ipm_step_vectors_batched).  Per Newton step there is exactly ONE collective: an all-reduce of an 8-double stats
vector (MAX of KKT residual / complementarity / inertia failures, MIN of step
lengths, SUM of active scenarios).  At the end, `gather_records` all-gathers
the per-scenario result records (scenario id, inertia, alpha_p, alpha_d,
residual norm, complementarity).  No data-path collective exists: scenarios
never exchange matrix data.
"""
from __future__ import annotations

import numpy as np

import torch
import torch.distributed as dist

from . import Plan
from .batch import BatchedKKTStep

REC = 8   # record: [scenario, pos, zero, neg, alpha_p, alpha_d, res_inf, compl_inf]


def partition(n_scenarios: int, world: int, rank: int):
    """Round-robin scenario ownership: rank r owns s with s % world == r."""
    return list(range(rank, n_scenarios, world))


def stats_vector(records: torch.Tensor, expected):
    """Local stopping-test statistics from a [S_local, REC] record tensor.
    Returns [max res_inf, max compl_inf, n_bad_inertia, -min alpha_p, -min alpha_d, n_active, 0, 0]
    so that ONE all_reduce(MAX) ... except n_active/n_bad which are SUMs: packed as a
    separate SUM slot (see global_stats)."""
    dev = records.device
    if records.numel() == 0:
        mx = torch.tensor([0.0, 0.0, 0.0, -1.0, -1.0], dtype=torch.float64, device=dev)
        sm = torch.tensor([0.0, 0.0], dtype=torch.float64, device=dev)
        return mx, sm
    ine = records[:, 1:4]
    exp = torch.tensor(expected, dtype=records.dtype, device=dev)
    bad = (ine != exp).any(dim=1).to(torch.float64)
    mx = torch.stack([records[:, 6].max(), records[:, 7].max(), bad.max(), (-records[:, 4]).max(),
                      (-records[:, 5]).max()])
    sm = torch.stack([bad.sum(), torch.tensor(float(records.shape[0]), dtype=torch.float64, device=dev)])
    return mx, sm


def global_stats(mx: torch.Tensor, sm: torch.Tensor, group=None):
    """The per-Newton-step global stopping test: one MAX and one SUM all-reduce
    of tiny vectors (NCCL over NVLink on GPUs, gloo in the CPU tests)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM, group=group)
    return dict(max_res_inf=float(mx[0]), max_compl_inf=float(mx[1]), any_bad_inertia=bool(mx[2] > 0),
                min_alpha_p=float(-mx[3]), min_alpha_d=float(-mx[4]), n_bad_inertia=int(sm[0]),
                n_scenarios=int(sm[1]))


def gather_records(records: torch.Tensor, n_scenarios: int, group=None):
    """All-gather per-scenario records and return them in global scenario order
    (rank-count independent: the same array for P = 1, 2, 4, 8)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        world = dist.get_world_size(group)
        cap = (n_scenarios + world - 1) // world
        buf = torch.full((cap, REC), -1.0, dtype=torch.float64, device=records.device)
        buf[: records.shape[0]] = records
        out = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(out, buf, group=group)
        allr = torch.cat(out).cpu().numpy()
    else:
        allr = records.cpu().numpy()
    allr = allr[allr[:, 0] >= 0]
    return allr[np.argsort(allr[:, 0], kind="stable")]


class ScopfBatch:
    """The local share of a SCOPF scenario batch on one GPU."""

    def __init__(self, base, scenario_fn, scenario_ids, sv_fn, device="cuda"):
        self.ids = list(scenario_ids)
        self.plan = Plan(base.n_s, base.n_d, base.m_E, base.m_I, base.rowptr, base.colidx)
        self.expected = (base.n_d, 0, base.m)
        n = len(self.ids)
        self.records = torch.zeros((n, REC), dtype=torch.float64, device=device)
        self.bt = None
        if n:
            def factory(i):
                p = scenario_fn(self.ids[i])
                return p, sv_fn(p, self.ids[i])
            self.bt = BatchedKKTStep((n, factory), plan=self.plan, device=device)
        self._ids_t = torch.tensor(self.ids, dtype=torch.float64, device=device)
        self.graph = self._capture() if n else None

    def _run(self, stream=None):
        self.bt.run(stream=stream)
        self._fill_records()

    def _capture(self):
        """ONE CUDA graph for the whole local batch (a Newton step is one graph launch)."""
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self._run(stream=side)                 # warm-up (workspaces, attributes)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._run(stream=torch.cuda.current_stream())
        return g

    def newton_step(self):
        """One Newton step's KKT work for every local scenario (one graph launch)."""
        if self.graph is not None:
            self.graph.replay()

    def results(self, i):
        return self.bt.results(i)

    def _fill_records(self):
        r, bt = self.records, self.bt
        r[:, 0] = self._ids_t
        r[:, 1:4] = bt.inertia.to(torch.float64)
        r[:, 4] = bt.vout[:, 0]
        r[:, 5] = bt.vout[:, 1]
        r[:, 6] = bt.vout[:, 6]
        r[:, 7] = bt.vout[:, 2]

    def stop_test(self, group=None):
        mx, sm = stats_vector(self.records, self.expected)
        return global_stats(mx, sm, group)
