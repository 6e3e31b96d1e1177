"""A batch of independent Newton-step KKT systems that share one sparsity
pattern (SCOPF contingency scenarios; north star: "independent
contingency KKT systems are batched per GPU"), resident on one GPU.

`BatchedKKTStep` stacks every per-scenario buffer ([B, ...] tensors, allocated
once) and issues the four batched C-ABI calls of include/mds.h in the paper's
order (Fig.1):
  mds_condense_batched -> mds_factor_batched -> mds_solve_batched
  -> ipm_step_vectors_batched
so one Newton step for all B scenarios is a fixed sequence of ~5 launches per
panel (for every scenario at once), not B per-scenario launch chains.  Per
scenario status / inertia / step-vector results land in [B]-shaped device
arrays; one failing scenario does not affect the others.  `run()` is
stream-ordered and CUDA-graph capturable.
"""
from __future__ import annotations

import numpy as np
import torch

from . import (Plan, DevPtr, ICParamsC, ICStateC, CondenseBatchedArgsC, FactorBatchedArgsC, ic_begin_batched,
               ic_step_batched, ic_graph_create, ic_graph_launch, ic_graph_destroy, condense_batched, factor_batched, solve_batched, step_vectors_batched,
               condense_workspace_size, factor_batched_workspace_size, solve_batched_workspace_size,
               step_vectors_batched_workspace_size)

VOUT = 16   # per-scenario step-vector result slots (6 + residual norms, padded)


class BatchedKKTStep:
    def __init__(self, probs, plan: Plan | None = None, svs=None, zero_tol=-1.0, device="cuda"):
        """probs: a sequence of MDS instances (same n_s, n_d, m_E, m_I and J_s
        pattern), or (B, factory) with factory(i) -> (prob, step_vectors or None),
        so that a large batch is loaded one scenario at a time; svs: optional K1
        step-vector inputs for (x_s, x_d), one per scenario."""
        if isinstance(probs, tuple) and callable(probs[1]):
            B, factory = int(probs[0]), probs[1]
        else:
            seq = list(probs)
            B = len(seq)
            factory = (lambda i: (seq[i], svs[i] if svs is not None else None))
        assert B >= 1
        p0, sv0 = factory(0)
        self.B = B
        self.n_s, self.n_d, self.m_E, self.m_I = int(p0.n_s), int(p0.n_d), int(p0.m_E), int(p0.m_I)
        self.m = self.m_E + self.m_I
        self.N = N = self.n_d + self.m
        self.plan = plan if plan is not None else Plan(self.n_s, self.n_d, self.m_E, self.m_I, p0.rowptr, p0.colidx)
        self.nnz = self.plan.nnz
        self.zero_tol = float(zero_tol)
        f64 = dict(dtype=torch.float64, device=device)
        n_s, n_d, m, m_I = self.n_s, self.n_d, self.m, self.m_I
        z = lambda w: torch.zeros((B, max(w, 1)), **f64)
        self.val, self.h_ss, self.sigma_s = z(self.nnz), z(n_s), z(n_s)
        self.ldh, self.ldj = max(n_d, 1), max(m, 1)
        self.H_dd, self.sigma_d, self.J_d, self.d_h = z(n_d * n_d), z(n_d), z(m * n_d), z(m_I)
        self.r = z(n_s + N)
        self.delta_w, self.delta_c = torch.zeros(B, **f64), torch.zeros(B, **f64)
        # outputs / intermediates
        self.ldm = N if N % 2 == 0 else N + 1           # 16-byte aligned columns (TMA)
        self.M = torch.empty((B, max(self.ldm * N, 2)), **f64)
        self.rhs = torch.empty((B, max(N, 1)), **f64)
        self.w = torch.empty((B, max(n_s, 1)), **f64)
        self.piv = torch.empty((B, max(2 * N, 1)), dtype=torch.int32, device=device)
        self.inertia = torch.zeros((B, 3), dtype=torch.int64, device=device)
        self.status = torch.zeros(B, dtype=torch.int32, device=device)
        self.anorm = torch.zeros(B, **f64)
        self.dirn = torch.empty((B, n_s + N), **f64)    # [dx_s | dx_d | dy_g | dy_h] per scenario
        self.cwork = torch.empty(condense_workspace_size(self.plan, B), dtype=torch.uint8, device=device)
        self.fwork = torch.empty(factor_batched_workspace_size(N, B), dtype=torch.uint8, device=device)
        self.swork = torch.empty(solve_batched_workspace_size(N, B), dtype=torch.uint8, device=device)
        self.nb = n_s + n_d
        self.sv = None
        if sv0 is not None:
            self._alloc_step_vectors()
        for i in range(B):
            p, sv = (p0, sv0) if i == 0 else factory(i)
            self.load(i, p, sv)

    def load(self, i, p, sv=None):
        """(Re)load scenario i's inputs (host arrays -> its rows of the batch)."""
        n_s, n_d, m, N = self.n_s, self.n_d, self.m, self.N

        def put(t, a, width):
            if width:
                t[i, :width] = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1))

        put(self.val, p.val, self.nnz)
        put(self.h_ss, p.h_ss, n_s)
        put(self.sigma_s, p.sigma_s, n_s)
        put(self.H_dd, np.asarray(p.H_dd).reshape(-1, order="F"), n_d * n_d)
        put(self.sigma_d, p.sigma_d, n_d)
        put(self.J_d, np.asarray(p.J_d).reshape(-1, order="F"), m * n_d)
        put(self.d_h, p.d_h, self.m_I)
        put(self.r, p.r, n_s + N)
        self.delta_w[i] = float(p.delta_w)
        self.delta_c[i] = float(p.delta_c)
        if sv is not None:
            if self.sv is None:
                self._alloc_step_vectors()
            nb = self.nb
            for k in ("x", "lo", "up", "zl", "zu", "dzl", "dzu"):
                self.sv[k][i, :nb] = torch.from_numpy(np.asarray(getattr(sv, k), dtype=np.float64))
            self.tau[i] = float(sv.tau)
            self.mu[i] = float(sv.mu)

    def _alloc_step_vectors(self):
        # rows padded to the direction's row width (n_s + N) so all 8 vectors share one stride
        B, n, W = self.B, self.nb, self.n_s + self.N
        dev = self.M.device
        self.sv = {k: torch.zeros((B, W), dtype=torch.float64, device=dev)
                   for k in ("x", "lo", "up", "zl", "zu", "dzl", "dzu")}
        self.tau = torch.zeros(B, dtype=torch.float64, device=dev)
        self.mu = torch.zeros(B, dtype=torch.float64, device=dev)
        self.vout = torch.zeros((B, VOUT), dtype=torch.float64, device=dev)
        self.sigma = torch.empty((B, W), dtype=torch.float64, device=dev)
        self.vwork = torch.empty(step_vectors_batched_workspace_size(n, B), dtype=torch.uint8, device=dev)

    # -- the hot path ------------------------------------------------------
    def run(self, stream=None):
        """One Newton step's KKT work for all B scenarios (no host sync)."""
        B, N, n_s = self.B, self.N, self.n_s
        self.status.zero_()
        strides = dict(val=self.val.shape[1], hss=self.h_ss.shape[1], sig=self.sigma_s.shape[1],
                       H=self.H_dd.shape[1], sd=self.sigma_d.shape[1], J=self.J_d.shape[1], dh=self.d_h.shape[1],
                       r=self.r.shape[1], M=self.M.shape[1], rhs=self.rhs.shape[1], w=self.w.shape[1])
        condense_batched(self.plan, B, self.val, self.h_ss, self.sigma_s, self.H_dd, self.ldh, self.sigma_d,
                         self.J_d, self.ldj, self.d_h, self.delta_w, self.delta_c, self.r, self.M, self.ldm,
                         self.rhs, self.w, self.anorm, self.status, self.cwork, strides, stream=stream)
        factor_batched(B, N, self.M, self.ldm, self.M.shape[1], self.piv, self.piv.shape[1], self.zero_tol,
                       self.inertia, self.status, self.fwork, anorm=self.anorm, stream=stream)
        # dxy of scenario s at dirn[s, n_s:], dx_s at dirn[s, :n_s]; r_xs at r[s, :n_s]
        dirn, W = self.dirn, self.dirn.shape[1]
        solve_batched(self.plan, B, N, self.M, self.ldm, self.M.shape[1], self.piv, self.piv.shape[1], self.rhs,
                      self.rhs.shape[1], self.val, self.val.shape[1], self.w, self.w.shape[1], self.r,
                      self.r.shape[1], DevPtr(dirn, n_s), W, DevPtr(dirn) if n_s else None, W, self.zero_tol,
                      self.fwork, self.status, self.swork, stream=stream)
        if self.sv is not None:
            s = self.sv
            step_vectors_batched(B, self.nb, W, s["x"], dirn, s["lo"], s["up"], s["zl"],
                                 s["zu"], s["dzl"], s["dzu"], 0.0, 0.0, self.vout, VOUT, self.sigma, self.status,
                                 self.vwork, tau_arr=self.tau, mu_arr=self.mu, res=(self.r,),
                                 res_str=((self.r.shape[1], self.r.shape[1]),), stream=stream)

    # -- inertia correction on the device (NEXT-1) ---------------------------
    def _ic_setup(self, params=None):
        if getattr(self, "_ic", None) is not None:
            return self._ic
        from .inertia import ICParams
        p = params or ICParams()
        B, dev = self.B, self.M.device
        st = dict(delta_w_last=torch.zeros(B, dtype=torch.float64, device=dev),
                  phase=torch.zeros(B, dtype=torch.int32, device=dev),
                  active=torch.ones(B, dtype=torch.int32, device=dev),
                  ntrial=torch.zeros(B, dtype=torch.int32, device=dev),
                  any_active=torch.zeros(1, dtype=torch.int32, device=dev))
        cst = ICStateC(self.delta_w.data_ptr(), self.delta_c.data_ptr(), st["delta_w_last"].data_ptr(),
                       st["phase"].data_ptr(), st["active"].data_ptr(), st["ntrial"].data_ptr(),
                       st["any_active"].data_ptr())
        cpar = ICParamsC(p.delta_w0, p.delta_w_min, p.delta_w_max, p.kappa_w_plus, p.kappa_w_plus_first,
                         p.kappa_w_minus, p.delta_c_bar, p.kappa_c)
        self._ic = dict(st, cstate=cst, cparams=cpar, graph=None, graph_mu=None)
        return self._ic

    def _strides(self):
        return dict(val=self.val.shape[1], hss=self.h_ss.shape[1], sig=self.sigma_s.shape[1], H=self.H_dd.shape[1],
                    sd=self.sigma_d.shape[1], J=self.J_d.shape[1], dh=self.d_h.shape[1], r=self.r.shape[1],
                    M=self.M.shape[1], rhs=self.rhs.shape[1], w=self.w.shape[1])

    def _trial(self, active, stream=None):
        B, N = self.B, self.N
        condense_batched(self.plan, B, self.val, self.h_ss, self.sigma_s, self.H_dd, self.ldh, self.sigma_d, self.J_d,
                         self.ldj, self.d_h, self.delta_w, self.delta_c, self.r, self.M, self.ldm, self.rhs, self.w,
                         self.anorm, self.status, self.cwork, self._strides(), stream=stream, active=active)
        factor_batched(B, N, self.M, self.ldm, self.M.shape[1], self.piv, self.piv.shape[1], self.zero_tol,
                       self.inertia, self.status, self.fwork, anorm=self.anorm, stream=stream, active=active)

    def factor_ic(self, mu, mode="graph", params=None, stream=None):
        """Condense + factor every scenario with the inertia correction of PAPER.md:161 on the
        device: failing scenarios (inertia != (n_d, 0, m)) are regularised with the next
        delta_w / delta_c of Algorithm IC and re-condensed / re-factored -- only they (mask) --
        until every scenario is accepted, failed (singular) or in error.  mode "graph": the
        whole loop is one CUDA graph with a conditional WHILE node (no host round trip);
        "host": the same kernels with one 4-byte read of any_active per round."""
        ic = self._ic_setup(params)
        B = self.B
        self.status.zero_()
        if mode == "graph":
            if ic["graph"] is None or ic["graph_mu"] != float(mu):
                if ic["graph"] is not None:
                    ic_graph_destroy(ic["graph"])
                self._trial(None, stream)          # warm-up (attributes, maps) outside capture
                ca = CondenseBatchedArgsC(B, self.val.data_ptr(), self.val.shape[1], self.h_ss.data_ptr(),
                                          self.h_ss.shape[1], self.sigma_s.data_ptr(), self.sigma_s.shape[1],
                                          self.H_dd.data_ptr(), self.ldh, self.H_dd.shape[1], self.sigma_d.data_ptr(),
                                          self.sigma_d.shape[1], self.J_d.data_ptr(), self.ldj, self.J_d.shape[1],
                                          self.d_h.data_ptr(), self.d_h.shape[1], self.r.data_ptr(), self.r.shape[1],
                                          self.M.data_ptr(), self.ldm, self.M.shape[1], self.rhs.data_ptr(),
                                          self.rhs.shape[1], self.w.data_ptr(), self.w.shape[1],
                                          self.anorm.data_ptr(), self.status.data_ptr(), self.cwork.data_ptr(),
                                          self.cwork.numel())
                fa = FactorBatchedArgsC(B, self.N, self.piv.data_ptr(), self.piv.shape[1], self.zero_tol,
                                        self.inertia.data_ptr(), self.fwork.data_ptr(), self.fwork.numel())
                torch.cuda.synchronize()
                ic["graph"] = ic_graph_create(self.plan, ca, fa, self.n_d, self.m, mu, ic["cparams"], ic["cstate"])
                ic["graph_mu"] = float(mu)
                self.status.zero_()
            ic_graph_launch(ic["graph"], stream)
        else:
            ic_begin_batched(B, ic["cstate"], stream)
            self._trial(None, stream)
            ic_step_batched(B, self.n_d, self.m, self.inertia, self.status, mu, ic["cparams"], ic["cstate"],
                            stream=stream)
            while int(ic["any_active"].item()) != 0:
                self._trial(ic["active"], stream)
                ic_step_batched(B, self.n_d, self.m, self.inertia, self.status, mu, ic["cparams"], ic["cstate"],
                                stream=stream)

    def ic_results(self):
        """(phase, ntrial, delta_w, delta_c) per scenario after factor_ic (synchronous)."""
        ic = self._ic
        return (ic["phase"].cpu().numpy(), ic["ntrial"].cpu().numpy(), self.delta_w.cpu().numpy(),
                self.delta_c.cpu().numpy())

    def finish(self, stream=None):
        """Solve + recovery + step vectors on the factorization left by factor_ic / run."""
        B, N, n_s = self.B, self.N, self.n_s
        dirn, W = self.dirn, self.dirn.shape[1]
        solve_batched(self.plan, B, N, self.M, self.ldm, self.M.shape[1], self.piv, self.piv.shape[1], self.rhs,
                      self.rhs.shape[1], self.val, self.val.shape[1], self.w, self.w.shape[1], self.r,
                      self.r.shape[1], DevPtr(dirn, n_s), W, DevPtr(dirn) if n_s else None, W, self.zero_tol,
                      self.fwork, self.status, self.swork, stream=stream)
        if self.sv is not None:
            s = self.sv
            step_vectors_batched(B, self.nb, W, s["x"], dirn, s["lo"], s["up"], s["zl"], s["zu"], s["dzl"],
                                 s["dzu"], 0.0, 0.0, self.vout, VOUT, self.sigma, self.status, self.vwork,
                                 tau_arr=self.tau, mu_arr=self.mu, res=(self.r,),
                                 res_str=((self.r.shape[1], self.r.shape[1]),), stream=stream)

    def capture(self, warmup=1):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.run(stream=s)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run(stream=torch.cuda.current_stream())
        return g

    # -- host views --------------------------------------------------------
    def results(self, i):
        """Scenario i's outputs as numpy arrays (synchronous; test / record use)."""
        torch.cuda.synchronize()
        n_s, N = self.n_s, self.N
        out = dict(inertia=tuple(int(v) for v in self.inertia[i].cpu()), dxy=self.dirn[i, n_s:n_s + N].cpu().numpy(),
                   dx_s=self.dirn[i, :n_s].cpu().numpy(), rhs_c=self.rhs[i, :N].cpu().numpy(),
                   w=self.w[i, :n_s].cpu().numpy(), status=int(self.status[i].item()),
                   anorm=float(self.anorm[i].item()))
        if self.sv is not None:
            v = self.vout[i].cpu().numpy()
            out["vec"] = dict(alpha_p=v[0], alpha_d=v[1], compl_inf=v[2], compl_sum=v[3], n_compl=int(v[4]),
                              first_bad=int(v[5]), res_inf=v[6])
            out["sigma"] = self.sigma[i, :self.nb].cpu().numpy()
        return out
