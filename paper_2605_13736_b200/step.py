"""One Newton step of the condensed-KKT hot path, resident on one GPU.

`KKTStep` owns every device buffer of a step (allocated once; nothing is
allocated inside `run`) and issues the four C-ABI calls in the paper's order
(Fig.1; §2.2-2.3):
  mds_condense -> mds_factor (inertia) -> mds_solve (+ dx_s recovery)
  -> ipm_step_vectors (fraction-to-boundary over (x_s, x_d), ||r||_inf).
`run()` is stream-ordered and CUDA-graph capturable (`capture()`).
"""
from __future__ import annotations

import numpy as np
import torch

from . import (Plan, condense, factor, solve, step_vectors, factor_workspace_size, solve_workspace_size,
               step_vectors_workspace_size, condense_workspace_size, raise_for)


def _dev(a, dtype=torch.float64, device="cuda"):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).to(device)


class DeviceProblem:
    """Device copies of one MDS instance's inputs (duck-typed: any object with
    the attributes of an Eq.(5) instance: n_s, n_d, m_E, m_I, rowptr, colidx,
    val, h_ss, sigma_s, H_dd (col-major), sigma_d, J_d (col-major), d_h,
    delta_w, delta_c, r)."""

    def __init__(self, prob, device="cuda", plan: Plan | None = None):
        self.n_s, self.n_d, self.m_E, self.m_I = int(prob.n_s), int(prob.n_d), int(prob.m_E), int(prob.m_I)
        self.m = self.m_E + self.m_I
        self.N = self.n_d + self.m
        self.plan = plan if plan is not None else Plan(self.n_s, self.n_d, self.m_E, self.m_I, prob.rowptr,
                                                       prob.colidx)
        one = np.zeros(1)
        self.val = _dev(prob.val if len(prob.val) else one, device=device)
        self.h_ss = _dev(prob.h_ss if self.n_s else one, device=device)
        self.sigma_s = _dev(prob.sigma_s if self.n_s else one, device=device)
        H = np.asarray(prob.H_dd)
        self.ldh = max(self.n_d, 1)
        self.H_dd = _dev(H.reshape(-1, order="F") if self.n_d else one, device=device)
        self.sigma_d = _dev(prob.sigma_d if self.n_d else one, device=device)
        J = np.asarray(prob.J_d)
        self.ldj = max(self.m, 1)
        self.J_d = _dev(J.reshape(-1, order="F") if (self.n_d and self.m) else one, device=device)
        self.d_h = _dev(prob.d_h if self.m_I else np.ones(1), device=device)
        self.delta_w, self.delta_c = float(prob.delta_w), float(prob.delta_c)
        self.r = _dev(prob.r, device=device)

    def host_bytes(self):
        """Bytes of per-step inputs (what an end-to-end call moves host->device)."""
        return sum(t.numel() * t.element_size() for t in (self.val, self.h_ss, self.sigma_s, self.H_dd,
                                                          self.sigma_d, self.J_d, self.d_h, self.r))


class KKTStep:
    def __init__(self, dprob: DeviceProblem, sv=None, zero_tol=-1.0, device="cuda"):
        self.p = dprob
        N, n_s, n_d = dprob.N, dprob.n_s, dprob.n_d
        self.N = N
        self.ldm = N if N % 2 == 0 else N + 1      # 16-byte aligned columns
        f64 = dict(dtype=torch.float64, device=device)
        self.M = torch.empty(max(self.ldm * N, 1), **f64)
        self.rhs = torch.empty(max(N, 1), **f64)
        self.w = torch.empty(max(n_s, 1), **f64)
        self.piv = torch.empty(max(2 * N, 1), dtype=torch.int32, device=device)
        self.inertia = torch.zeros(3, dtype=torch.int64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.fwork = torch.empty(factor_workspace_size(N), dtype=torch.uint8, device=device)
        self.cwork = torch.empty(condense_workspace_size(dprob.plan), dtype=torch.uint8, device=device)
        self.anorm = torch.zeros(1, dtype=torch.float64, device=device)   # ||M||_inf (a3, fused into a2)
        self.swork = torch.empty(solve_workspace_size(N), dtype=torch.uint8, device=device)
        # direction laid out [dx_s | dx_d | dy_g | dy_h] so (dx_s, dx_d) is contiguous
        self.dirn = torch.empty(n_s + N + 1, **f64)
        self.dx_s = self.dirn[:n_s] if n_s else None
        self.dxy = self.dirn[n_s:n_s + N]
        self.zero_tol = float(zero_tol)
        self.nb = n_s + n_d
        self.sv = None
        if sv is not None:
            self.set_step_vectors(sv)

    def set_step_vectors(self, sv):
        """K1 inputs for the (x_s, x_d) primal block: x, lo, up, zl, zu, dzl, dzu (host arrays of length
        n_s+n_d), tau, mu.  The primal direction dx is the solve's output."""
        n = self.nb
        assert len(sv.x) == n, "step vectors must cover (x_s, x_d)"
        d = lambda a: _dev(a)
        self.sv = dict(x=d(sv.x), lo=d(sv.lo), up=d(sv.up), zl=d(sv.zl), zu=d(sv.zu), dzl=d(sv.dzl),
                       dzu=d(sv.dzu), tau=float(sv.tau), mu=float(sv.mu))
        self.vout = torch.zeros(16, dtype=torch.float64, device=self.M.device)
        self.sigma = torch.empty(max(n, 1), dtype=torch.float64, device=self.M.device)
        self.vwork = torch.zeros(step_vectors_workspace_size(n), dtype=torch.uint8, device=self.M.device)

    # -- the hot path ------------------------------------------------------
    def run(self, stream=None, sync_inertia=False, marks=None):
        """One Newton step.  `marks`: optional list of 5 CUDA events recorded on the
        stream between the four calls (wall-clock phase timing)."""
        ev = (lambda i: marks[i].record(stream) if stream is not None else marks[i].record()) if marks else \
            (lambda i: None)
        ine = self.factor_phase(stream, sync_inertia, ev)
        self.finish_phase(stream, ev)
        return ine

    def factor_phase(self, stream=None, sync_inertia=False, ev=None):
        """mds_condense (with the problem's current delta_w, delta_c) + mds_factor.
        Returns the inertia triple when sync_inertia (the only host sync), else None."""
        p = self.p
        ev = ev or (lambda i: None)
        self.status.zero_()
        ev(0)
        condense(p.plan, p.val, p.h_ss, p.sigma_s, p.H_dd, p.ldh, p.sigma_d, p.J_d, p.ldj, p.d_h, p.delta_w,
                 p.delta_c, p.r, self.M, self.ldm, self.rhs, self.w, self.status, stream, anorm_out=self.anorm,
                 work=self.cwork)
        ev(1)
        ine = factor(self.N, self.M, self.ldm, self.piv, self.zero_tol, self.inertia, self.status, self.fwork,
                     sync=sync_inertia, stream=stream, anorm=self.anorm)
        ev(2)
        return ine

    def finish_phase(self, stream=None, ev=None):
        """mds_solve (+ dx_s recovery) and ipm_step_vectors on the factor left by factor_phase."""
        p = self.p
        ev = ev or (lambda i: None)
        solve(p.plan, self.N, self.M, self.ldm, self.piv, self.rhs, p.val, self.w, p.r[:p.n_s] if p.n_s else None,
              self.dxy, self.dx_s, self.zero_tol, self.fwork, self.status, self.swork, stream)
        ev(3)
        if self.sv is not None:
            s = self.sv
            step_vectors(self.nb, s["x"], self.dirn[:self.nb], s["lo"], s["up"], s["zl"], s["zu"], s["dzl"],
                         s["dzu"], s["tau"], s["mu"], self.vout, self.sigma, self.status, self.vwork,
                         res=(p.r,), stream=stream)
        ev(4)

    def capture(self, warmup=1):
        """CUDA-graph of run() (no host sync inside)."""
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

    def capture_phases(self, warmup=1):
        """CUDA graphs of factor_phase() (with the problem's current delta_w, delta_c, which
        the graph bakes in) and of finish_phase(): the two halves of run() around the
        inertia check."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.run(stream=s)
        torch.cuda.current_stream().wait_stream(s)
        gf, gs = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(gf):
            self.factor_phase(stream=torch.cuda.current_stream())
        with torch.cuda.graph(gs):
            self.finish_phase(stream=torch.cuda.current_stream())
        return gf, gs

    # -- host views --------------------------------------------------------
    def check_status(self):
        st = int(self.status.item())
        if st != 0:
            raise_for(st, "KKT step")

    def M_host(self):
        """M (or LD after factor) as a numpy (N x N) array, A[i, j] = M[i + j*ldm]."""
        N = self.N
        return self.M[: self.ldm * N].view(N, self.ldm)[:, :N].cpu().numpy().T

    def results(self):
        torch.cuda.synchronize()
        out = dict(inertia=tuple(int(v) for v in self.inertia.cpu()), dxy=self.dxy.cpu().numpy(),
                   dx_s=(self.dx_s.cpu().numpy() if self.dx_s is not None else np.zeros(0)),
                   rhs_c=self.rhs[: self.N].cpu().numpy(), w=self.w[: self.p.n_s].cpu().numpy(),
                   status=int(self.status.item()))
        if self.sv is not None:
            v = self.vout.cpu().numpy()
            out["vec"] = dict(alpha_p=v[0], alpha_d=v[1], compl_inf=v[2], compl_sum=v[3], n_compl=int(v[4]),
                              first_bad=int(v[5]), res_inf=v[6])
            out["sigma"] = self.sigma[: self.nb].cpu().numpy()
        return out


class HostPipeline:
    """Newton steps whose inputs live in HOST (pinned) memory, end to end: each step
    uploads its inputs (the DeviceProblem arrays), runs the hot path, and downloads
    its results (dx, inertia, step-vector scalars).  The copies of step i+1 and
    step i-1 run on a copy stream while step i computes: two device input sets and
    two `KKTStep`s (one plan) alternate, so the PCIe traffic overlaps the factorization
    instead of adding to it.  Stream order alone carries every dependency (no host
    synchronisation inside `run`)."""

    IN = ("val", "h_ss", "sigma_s", "H_dd", "sigma_d", "J_d", "d_h", "r")

    def __init__(self, prob, sv=None, device="cuda", use_graph=True):
        d0 = DeviceProblem(prob, device)
        self.dp = [d0, DeviceProblem(prob, device, plan=d0.plan)]
        self.st = [KKTStep(dp, sv=sv, device=device) for dp in self.dp]
        self.graphs = [s.capture() for s in self.st] if use_graph else None
        self.comp = torch.cuda.Stream(device=device)
        self.copy = torch.cuda.Stream(device=device)
        self.up = [torch.cuda.Event() for _ in range(2)]
        self.done = [torch.cuda.Event() for _ in range(2)]

    def pinned_inputs(self):
        """A pinned host copy of the current inputs (one set; the caller may refill it)."""
        return [torch.empty(getattr(self.dp[0], k).shape, dtype=torch.float64, pin_memory=True).copy_(
            getattr(self.dp[0], k).cpu()) for k in self.IN]

    def outputs(self, k):
        s = self.st[k]
        o = [s.dxy, s.inertia]
        if s.dx_s is not None:
            o.append(s.dx_s)
        if s.sv is not None:
            o.append(s.vout)
        return o

    def pinned_outputs(self):
        return [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in self.outputs(0)]

    def bytes_per_step(self, host_in, host_out):
        return (sum(t.numel() * t.element_size() for t in host_in),
                sum(t.numel() * t.element_size() for t in host_out))

    def _upload(self, k, host_in):
        with torch.cuda.stream(self.copy):
            self.copy.wait_event(self.done[k])       # slot k's previous step has consumed its inputs
            for name, h in zip(self.IN, host_in):
                getattr(self.dp[k], name).copy_(h, non_blocking=True)
            self.up[k].record(self.copy)

    def run(self, steps, host_in, host_out, start=None, end=None):
        """`steps` Newton steps, each from `host_in` (pinned, `pinned_inputs()` layout) with the
        results of each step written to `host_out` (`pinned_outputs()`).  `start` / `end`:
        optional CUDA events recorded around the whole sequence (on the copy stream)."""
        cur = torch.cuda.current_stream()
        self.copy.wait_stream(cur)
        self.comp.wait_stream(cur)
        if start is not None:
            start.record(self.copy)
        self._upload(0, host_in)
        for i in range(steps):
            k = i & 1
            self.comp.wait_event(self.up[k])
            with torch.cuda.stream(self.comp):
                if self.graphs is not None:
                    self.graphs[k].replay()
                else:
                    self.st[k].run(stream=self.comp)
                self.done[k].record(self.comp)
            if i + 1 < steps:
                self._upload(k ^ 1, host_in)          # step i+1's inputs while step i computes
            with torch.cuda.stream(self.copy):
                self.copy.wait_event(self.done[k])
                for h, d in zip(host_out, self.outputs(k)):
                    h.copy_(d, non_blocking=True)
        if end is not None:
            end.record(self.copy)
        cur.wait_stream(self.copy)
        cur.wait_stream(self.comp)
