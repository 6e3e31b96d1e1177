"""Security-constrained OPF scenario batching (north star:
"Independent contingency KKT systems are batched per GPU across the 8xB200
box, and NCCL over NVLink is used only to gather per-scenario results and the
global stopping test").

One process per GPU.  Rank r owns the scenarios s with s % P == r (round-robin,
so scenarios that converge at different iteration counts stay balanced).  Each
scenario is one `KKTStep` (all share the pattern plan); the local scenarios run
concurrently on a pool of CUDA streams, each replaying its own CUDA graph.  Per
Newton step there is exactly ONE collective: an all-reduce of an 8-double stats
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

from . import Plan, set_grid_cap
from .step import DeviceProblem, KKTStep

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

    def __init__(self, base, scenario_fn, scenario_ids, sv_fn, n_streams=8, device="cuda", grid_cap=0):
        self.ids = list(scenario_ids)
        self.plan = Plan(base.n_s, base.n_d, base.m_E, base.m_I, base.rowptr, base.colidx)
        self.expected = (base.n_d, 0, base.m)
        n = len(self.ids)
        self.records = torch.zeros((n, REC), dtype=torch.float64, device=device)
        self.steps = []
        for i, s in enumerate(self.ids):
            prob = scenario_fn(s)
            st = KKTStep(DeviceProblem(prob, plan=self.plan), sv=sv_fn(prob, s))
            self.steps.append(st)
        self.streams = [torch.cuda.Stream() for _ in range(max(1, min(n_streams, n)))]
        # concurrent factorizations share the SMs: cap each persistent update grid
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        cap = int(grid_cap) or max(8, sms // len(self.streams))
        # (a capped grid also selects the factorization's concurrent launch structure -- no
        #  one-launch tail panels -- so a scenario's bits depend on the cap, never on the stream
        #  count, the rank or the other scenarios)
        self.grid_cap = cap if len(self.streams) > 1 else 0
        set_grid_cap(self.grid_cap)
        self._ids_t = torch.tensor(self.ids, dtype=torch.float64, device=device)
        self.graph = self._capture_all()
        set_grid_cap(0)

    def _run_all(self):
        cur = torch.cuda.current_stream()
        for s in self.streams:
            s.wait_stream(cur)
        for i, st in enumerate(self.steps):
            s = self.streams[i % len(self.streams)]
            with torch.cuda.stream(s):
                st.run(stream=s)
        for s in self.streams:
            cur.wait_stream(s)
        self._fill_records()

    def _capture_all(self):
        """ONE CUDA graph for the whole local batch: the capture forks onto the
        stream pool (one branch per stream) and joins back, so a Newton step is a
        single graph launch."""
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self._run_all()                       # warm-up (workspaces, look-ahead contexts)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._run_all()
        return g

    def newton_step(self):
        """One Newton step's KKT work for every local scenario (one graph launch)."""
        self.graph.replay()

    def _fill_records(self):
        r = self.records
        if not self.steps:
            return
        r[:, 0] = self._ids_t
        r[:, 1:4] = torch.stack([st.inertia for st in self.steps]).to(torch.float64)
        v = torch.stack([st.vout for st in self.steps])
        r[:, 4] = v[:, 0]
        r[:, 5] = v[:, 1]
        r[:, 6] = v[:, 6]
        r[:, 7] = v[:, 2]

    def stop_test(self, group=None):
        mx, sm = stats_vector(self.records, self.expected)
        return global_stats(mx, sm, group)
