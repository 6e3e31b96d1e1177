"""Distributed LDL^T of ONE condensed KKT system across GPUs (SURVEY.md §8(f)
NEXT-4).  The paper's implementation is single-GPU ("does not support
distributed memory parallelism"; larger grids are future work,
PAPER.md:100); this is the B200-native extension for an N beyond one GPU's
memory: one process per GPU, torch.distributed (NCCL over NVLink/NVSwitch; gloo
in the CPU-only / one-GPU tests) for the exchanges, every arithmetic step in the
C-ABI kernels of csrc/dist.cu (and mds_factor / mds_solve for the exact phase).

Layout: the lower triangle of M in 64-column panels, panel g owned by rank
g mod P (1-D block-cyclic), each rank storing its panels full height
(`DistLDLT.C`: column-major, ld = N, global row index).  Factor, panel by panel
(right-looking, the Bunch-Kaufman speculative-panel scheme of the single-GPU
factor, R19):

  owner(p): mds_dist_panel -- unpivoted LDL^T of the panel + the BK 1x1
            acceptance test |d_j| >= alpha colmax_j of every column;
  all:      broadcast of the accepted flag, then of the panel's (L, W = L D);
            mds_dist_update on the rank's later panels (C -= L W^T, DMMA).

The first panel that fails the test ends the distributed phase: the Schur
complement S of everything before it (all panels from it on) is gathered on the
panel's owner and factored there by mds_factor -- exact Bunch-Kaufman with
interchanges and 2x2 pivots, the same decisions the single-GPU factor takes from
that column on.  inertia(M) = inertia(D_1) + inertia(S) (Haynsworth, PAPER.md:191;
zero band tol = N eps ||M||_inf of the whole M, reading R4).  Quasi-definite IPM
matrices (the accepted-every-panel case) never leave the distributed phase.

Solve (block form, M = [L1 0; L21 I] diag(D1, S) [L1^T L21^T; 0 I]):
  forward  y_p = L_pp^-1 (b_p - sum_r acc_r[p]) per panel (all-reduce of the 64
           partial sums; the owner then adds L(:, p) y_p to its accumulator);
  trailing x_2 = S^-1 (b_2 - sum_r acc_r[2]) on the exact-phase rank (mds_solve),
           broadcast;
  backward x_p = L_pp^-T (y_p / d_p - L(rows below, p)^T x) per panel, owner
           computes, broadcasts x_p.
Host logic only; no arithmetic of the method here.
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist

from . import (DevPtr, dist_panel, dist_update, dist_trsv64, dist_gemv_n, dist_gemv_t, dist_rowabs, factor,
               factor_workspace_size, solve, solve_workspace_size)
from .errors import SingularError, raise_for

DB = 64
EPS = float(np.finfo(np.float64).eps)


def panel_owner(g: int, world: int) -> int:
    """Owner rank of panel g (1-D block-cyclic)."""
    return g % world


def local_panels(npanel: int, rank: int, world: int):
    """Global panel indices of `rank`, ascending (local index = position)."""
    return list(range(rank, npanel, world))


def panel_span(g: int, N: int):
    """(first column, width) of panel g."""
    k0 = g * DB
    return k0, min(DB, N - k0)


class _Comm:
    """Collectives on CUDA tensors: direct for NCCL, staged through host memory for gloo."""

    def __init__(self, group=None):
        self.group = group
        self.on = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.on else 0
        self.world = dist.get_world_size(group) if self.on else 1
        self.stage = self.on and dist.get_backend(group) != "nccl"

    def bcast(self, t, src):
        if self.world == 1:
            return t
        if self.stage:
            h = t.cpu()
            dist.broadcast(h, src=self._g(src), group=self.group)
            t.copy_(h)
        else:
            dist.broadcast(t, src=self._g(src), group=self.group)
        return t

    def allsum(self, t):
        if self.world == 1:
            return t
        if self.stage:
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def _g(self, r):
        return dist.get_global_rank(self.group, r) if (self.on and self.group is not None) else r


class DistLDLT:
    """One N x N symmetric matrix distributed over the ranks of `group` (see the
    module docstring).  load_columns / load_full fill the local panels; factor()
    and solve(b) are collective (every rank calls them)."""

    def __init__(self, N: int, group=None, device=None, zero_tol: float = -1.0):
        self.comm = _Comm(group)
        self.rank, self.world = self.comm.rank, self.comm.world
        self.N = int(N)
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.np = max(1, math.ceil(self.N / DB))
        self.mine = local_panels(self.np, self.rank, self.world)
        nq = len(self.mine)
        # local panels: [nq * 64, N] row-major == column-major N x (nq * 64), ld = N
        self.C = torch.zeros((max(nq, 1) * DB, self.N), dtype=torch.float64, device=self.dev)
        self.kq = torch.tensor([panel_span(g, self.N)[0] for g in self.mine] or [0], dtype=torch.int64,
                               device=self.dev)
        self.wq = torch.tensor([panel_span(g, self.N)[1] for g in self.mine] or [0], dtype=torch.int32,
                               device=self.dev)
        self.zero_tol = float(zero_tol)
        self.d = {}              # global panel -> device d (owner only)
        self.pf = self.np        # first panel of the exact phase (np: none)
        self.S = None            # exact phase (on its rank): factored Schur complement
        self.inertia = None

    # -- data -------------------------------------------------------------
    def local_index(self, g: int) -> int:
        return (g - self.rank) // self.world

    def load_columns(self, g: int, cols):
        """Columns of panel g (device or host array [N, width], column j of M in column j)."""
        k0, w = panel_span(g, self.N)
        q = self.local_index(g)
        src = torch.as_tensor(np.ascontiguousarray(np.asarray(cols).T) if not torch.is_tensor(cols) else cols.T,
                              dtype=torch.float64)
        self.C[q * DB:q * DB + w, :] = src.to(self.dev)

    def load_full(self, M):
        """Every rank takes its panels' columns of the full (host) matrix M."""
        for g in self.mine:
            k0, w = panel_span(g, self.N)
            self.load_columns(g, np.asarray(M)[:, k0:k0 + w])

    def _panel_ptr(self, g: int, row: int = 0):
        return DevPtr(self.C, self.local_index(g) * DB * self.N + row)

    # -- factor -----------------------------------------------------------
    def factor(self):
        N, comm = self.N, self.comm
        nq = len(self.mine)
        # ||M||_inf (fixed order per rank, summed over ranks) -> the zero band
        rs = torch.zeros(N, dtype=torch.float64, device=self.dev)
        if nq:
            dist_rowabs(N, self.C, N, self.kq, self.wq, nq, rs)
        comm.allsum(rs)
        anorm = float(rs.max().item()) if N else 0.0
        self.tol = self.zero_tol if self.zero_tol >= 0 else N * EPS * anorm
        ine = torch.zeros(3, dtype=torch.int64, device=self.dev)
        acc = torch.zeros(1, dtype=torch.int32, device=self.dev)
        Lb = torch.empty((DB, N), dtype=torch.float64, device=self.dev)   # broadcast panel (L), ld = n
        Wb = torch.empty((DB, N), dtype=torch.float64, device=self.dev)
        d = torch.empty(DB, dtype=torch.float64, device=self.dev)
        cmax = torch.empty(DB, dtype=torch.float64, device=self.dev)
        parts = torch.empty((max(1, math.ceil(N / 128)), DB), dtype=torch.float64, device=self.dev)
        self.pf = self.np
        for p in range(self.np):
            k0, nb = panel_span(p, N)
            n = N - k0
            owner = panel_owner(p, self.world)
            if self.rank == owner:   # (L, W packed in the broadcast buffers, ld = n; the panel is untouched)
                dist_panel(n, nb, self._panel_ptr(p, k0), N, DevPtr(Lb), DevPtr(Wb), n, d, cmax, parts,
                           parts.shape[0], self.tol, acc, ine)
            comm.bcast(acc, owner)
            if int(acc.item()) == 0:
                self.pf = p
                break
            if self.rank == owner:   # accepted: the panel's storage becomes its L (for the solve)
                self.d[p] = d[:nb].clone()
                q = self.local_index(p)
                self.C[q * DB:q * DB + nb, k0:] = Lb.view(-1)[:nb * n].view(nb, n)
            lb = Lb.view(-1)[:nb * n]
            wb = Wb.view(-1)[:nb * n]
            comm.bcast(lb, owner)
            comm.bcast(wb, owner)
            later = [i for i, g in enumerate(self.mine) if g > p]
            if later:
                q0 = later[0]
                dist_update(N, k0, nb, DevPtr(Lb), DevPtr(Wb), n, DevPtr(self.C, q0 * DB * N), N,
                            DevPtr(self.kq, q0), DevPtr(self.wq, q0), len(later), N - self.mine[q0] * DB)
        if self.pf < self.np:
            self._exact_phase(ine)
        comm.allsum(ine)
        self.inertia = tuple(int(v) for v in ine.cpu())
        return self.inertia

    def _exact_phase(self, ine):
        """Gather the Schur complement (panels pf..) on owner(pf); mds_factor there."""
        N, comm = self.N, self.comm
        kf = self.pf * DB
        n2 = N - kf
        root = panel_owner(self.pf, self.world)
        S = torch.zeros((n2, n2), dtype=torch.float64, device=self.dev) if self.rank == root else None
        buf = torch.empty((DB, n2), dtype=torch.float64, device=self.dev)
        for g in range(self.pf, self.np):
            k0, w = panel_span(g, N)
            o = panel_owner(g, self.world)
            b = buf[:w]
            if self.rank == o:
                q = self.local_index(g)
                b.copy_(self.C[q * DB:q * DB + w, kf:])
            comm.bcast(b, o)
            if self.rank == root:
                S[k0 - kf:k0 - kf + w, :] = b       # rows of S (row-major) = columns of the col-major S
        if self.rank == root:
            piv = torch.empty(2 * n2, dtype=torch.int32, device=self.dev)
            ine2 = torch.zeros(3, dtype=torch.int64, device=self.dev)
            status = torch.zeros(1, dtype=torch.int32, device=self.dev)
            fwork = torch.empty(factor_workspace_size(n2), dtype=torch.uint8, device=self.dev)
            factor(n2, S, n2, piv, self.tol, ine2, status, fwork, sync=True)
            st = int(status.item())
            if st != 0:
                raise_for(st, "distributed LDL^T: exact phase")
            ine += ine2
            self.S = (S, piv, fwork)

    # -- solve ------------------------------------------------------------
    def solve(self, b):
        """x = M^-1 b (b: device vector, the same on every rank); x on every rank."""
        N, comm = self.N, self.comm
        b = b.to(self.dev, torch.float64)
        acc = torch.zeros(N, dtype=torch.float64, device=self.dev)
        x = torch.zeros(N, dtype=torch.float64, device=self.dev)
        y = {}
        bad = torch.zeros(1, dtype=torch.int32, device=self.dev)
        for p in range(self.pf):
            k0, nb = panel_span(p, N)
            owner = panel_owner(p, self.world)
            s = acc[k0:k0 + nb].clone()
            comm.allsum(s)
            if self.rank == owner:
                yp = (b[k0:k0 + nb] - s).contiguous()
                dist_trsv64(nb, self._panel_ptr(p, k0), N, yp, 0)
                dist_gemv_n(k0 + nb, N, nb, self._panel_ptr(p), N, yp, acc)
                dp = self.d[p]
                if bool((dp.abs() <= self.tol).any()):
                    bad.fill_(1)
                y[p] = yp / dp
        if self.pf < self.np:
            kf = self.pf * DB
            s2 = acc[kf:].clone()
            comm.allsum(s2)
            root = panel_owner(self.pf, self.world)
            x2 = x[kf:]
            if self.rank == root:
                S, piv, fwork = self.S
                n2 = N - kf
                rhs = (b[kf:] - s2).contiguous()
                out = torch.empty(n2, dtype=torch.float64, device=self.dev)
                st = torch.zeros(1, dtype=torch.int32, device=self.dev)
                swork = torch.empty(solve_workspace_size(n2), dtype=torch.uint8, device=self.dev)
                solve(None, n2, S, n2, piv, rhs, None, None, None, out, None, self.tol, fwork, st, swork)
                if int(st.item()) != 0:
                    bad.fill_(1)
                x2.copy_(out)
            comm.bcast(x2, root)
        comm.allsum(bad)
        if int(bad.item()) != 0:
            raise SingularError("distributed LDL^T solve: zero pivot (|d| <= tol)")
        for p in range(self.pf - 1, -1, -1):
            k0, nb = panel_span(p, N)
            owner = panel_owner(p, self.world)
            xp = x[k0:k0 + nb]
            if self.rank == owner:
                t = torch.empty(nb, dtype=torch.float64, device=self.dev)
                dist_gemv_t(k0 + nb, N, nb, self._panel_ptr(p), N, x, t)
                z = (y[p] - t).contiguous()
                dist_trsv64(nb, self._panel_ptr(p, k0), N, z, 1)
                xp.copy_(z)
            comm.bcast(xp, owner)
        return x
