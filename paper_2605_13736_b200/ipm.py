"""The interior-point loop around the hot path, on the device (SURVEY.md §8(f)
NEXT-2; PAPER.md:134-140 filter line search, Fig.1).

`IPMSolver` runs the primal-dual filter line-search IPM of DESIGN.md reading R23
on a convex QP in MDS form (duck-typed: base (an Eq.(5) instance with the
Hessian and Jacobian blocks), c, g_E, h_l, h_u, lo, up, x_star).  Every Newton iteration is the
paper's hot path through the C-ABI -- mds_condense, mds_factor (inertia,
corrected by `InertiaCorrection` when needed), mds_solve, ipm_step_vectors --
plus the IPM vector kernels (ipm_rhs, ipm_directions, ipm_reduce, ipm_apply)
and two K0 products (mds_kkt_residual).  Barrier-parameter, filter and
step-acceptance decisions are host control logic on a few scalars per
iteration (the error norms, the line-search terms, one pair per trial point);
all vector arithmetic runs in the library's kernels.  The iterate never leaves
the GPU.  The initial point is set up once with torch elementwise ops
(x = x_star, s = J_I x_star, bound duals mu0 / gap, y = 0).
"""
from __future__ import annotations

import time

import numpy as np
import torch

from . import (factor_stats, ipm_apply, ipm_directions, ipm_reduce, ipm_rhs, ipm_workspace_size, kkt_residual,
               kkt_residual_workspace_size,
               step_vectors, step_vectors_workspace_size, raise_for)
from .inertia import InertiaCorrection
from .step import DeviceProblem, KKTStep

INF = 1e20
OPTS = dict(tol=1e-8, mu0=0.1, max_iter=200, tau_min=0.99, kappa_mu=0.2, theta_mu=1.5, kappa_eps=10.0,
            gamma_theta=1e-5, gamma_phi=1e-5, s_theta=1.1, s_phi=2.3, eta_phi=1e-4, delta=1.0,
            kappa_Sigma=1e10, alpha_min_frac=1e-14)


class IPMSolver:
    def __init__(self, qp, opts=None, device="cuda", use_graph=True):
        self.o = dict(OPTS, **(opts or {}))
        b = qp.base
        self.n_s, self.n_d, self.m_E, self.m_I = b.n_s, b.n_d, b.m_E, b.m_I
        n, m, m_I = b.n_s + b.n_d, b.m_E + b.m_I, b.m_I
        self.n, self.m = n, m
        f64 = dict(dtype=torch.float64, device=device)
        dev = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(device)
        self.dp = dp = DeviceProblem(b, device=device)
        # Newton-system inputs written by ipm_rhs each iteration: sigma over P (its slack tail
        # is D_h) and the Eq.(5) right-hand side r; the DeviceProblem views them in place
        self.sigma = torch.zeros(n + m_I + 1, **f64)
        self.r = torch.zeros(n + m + 1, **f64)
        dp.sigma_s = self.sigma[:b.n_s] if b.n_s else dp.sigma_s
        dp.sigma_d = self.sigma[b.n_s:n] if b.n_d else dp.sigma_d
        dp.d_h = self.sigma[n:n + m_I] if m_I else dp.d_h
        dp.r = self.r[:n + m]
        dp.delta_w = dp.delta_c = 0.0
        self.step = KKTStep(dp, device=device)
        self.ic = InertiaCorrection(self.step, use_graph=use_graph)
        # K0 = the Eq.(5) blocks with sigma = delta = 0, D_y = 0 (for (H x + J^T y, J x) products)
        self.zero_s = torch.zeros(max(b.n_s, 1), **f64)
        self.zero_d = torch.zeros(max(b.n_d, 1), **f64)
        self.inf_h = torch.full((max(m_I, 1),), float("inf"), **f64)
        self.kwork = torch.empty(kkt_residual_workspace_size(dp.plan), dtype=torch.uint8, device=device)
        # problem data over the P = [x | s] layout
        self.c = dev(qp.c)
        self.g_E = dev(qp.g_E) if b.m_E else torch.zeros(1, **f64)
        self.lo = dev(np.concatenate([qp.lo, qp.h_l]))
        self.up = dev(np.concatenate([qp.up, qp.h_u]))
        # iterate
        self.P = torch.zeros(n + m_I, **f64)
        self.zl = torch.zeros(n + m_I, **f64)
        self.zu = torch.zeros(n + m_I, **f64)
        self.y = torch.zeros(max(m, 1), **f64)
        self.xy = torch.zeros(n + m, **f64)
        # work vectors
        self.Kxy = torch.zeros(n + m, **f64)
        self.Kd = torch.zeros(n + m, **f64)
        self.dx0 = torch.zeros(n + m, **f64)
        self.q = torch.zeros(max(m_I, 1), **f64)
        self.res_d = torch.zeros(n + m_I, **f64)
        self.res_p = torch.zeros(max(m, 1), **f64)
        self.dP = torch.zeros(n + m_I, **f64)
        self.dzl = torch.zeros(n + m_I, **f64)
        self.dzu = torch.zeros(n + m_I, **f64)
        self.vout = torch.zeros(16, **f64)
        self.vstatus = torch.zeros(1, dtype=torch.int32, device=device)
        self.vwork = torch.zeros(step_vectors_workspace_size(n + m_I), dtype=torch.uint8, device=device)
        self.rwork = torch.zeros(ipm_workspace_size(n, m_I), dtype=torch.uint8, device=device)
        self.red = torch.zeros((3, 8), **f64)
        self._init_point(qp)

    def reset(self, qp):
        """Back to the initial point of `qp` (same problem data), keeping the device buffers
        and the captured graphs: a second trajectory from the same start."""
        self._init_point(qp)
        self.ic.delta_w_last = 0.0

    # -- K0 product: out = (H v_x + J^T v_y, J v_x)
    def _k0(self, v, out):
        dp = self.dp
        kkt_residual(dp.plan, dp.val, dp.h_ss, self.zero_s, dp.H_dd, dp.ldh, self.zero_d, dp.J_d, dp.ldj, self.inf_h,
                     0.0, 0.0, v, None, out, work=self.kwork)

    def _init_point(self, qp):
        n, m_E, m_I, mu0 = self.n, self.m_E, self.m_I, self.o["mu0"]
        self.xy[:n] = torch.as_tensor(np.asarray(qp.x_star, dtype=np.float64)).to(self.xy.device)
        self.xy[n:] = 0.0
        self._k0(self.xy, self.Kxy)
        self.P[:n] = self.xy[:n]
        self.P[n:] = self.Kxy[n + m_E:]                       # s = J_I x_star
        fl, fu = self.lo.abs() < INF, self.up.abs() < INF
        gl, gu = self.P - self.lo, self.up - self.P
        if bool(((gl <= 0) & fl).any()) or bool(((gu <= 0) & fu).any()):
            raise_for(-6, "IPM initial point")
        self.zl = torch.where(fl, mu0 / torch.where(fl, gl, 1.0), 0.0).contiguous()
        self.zu = torch.where(fu, mu0 / torch.where(fu, gu, 1.0), 0.0).contiguous()
        self.y.zero_()

    def solve(self, log=None):
        """Run to e_0 <= tol.  Returns dict(status, iterations, mu, e0, history, seconds, newton_ms)."""
        o = self.o
        n, m, m_E, m_I = self.n, self.m, self.m_E, self.m_I
        mu = o["mu0"]
        filt = []
        hist = []
        status = "MaxIter"
        e0 = float("nan")
        newton_ms = []
        torch.cuda.synchronize()
        t_start = time.perf_counter()
        it = 0
        for it in range(o["max_iter"] + 1):
            self._k0(self.xy, self.Kxy)
            ipm_rhs(n, m_E, m_I, self.Kxy, self.c, self.g_E, self.P, self.lo, self.up, self.zl, self.zu, self.y, mu,
                    self.sigma, self.r, self.q, self.res_d, self.res_p)
            ipm_reduce(0, n, m_E, m_I, self.red[0], self.rwork, self.P, self.lo, self.up, zl=self.zl, zu=self.zu,
                       res_d=self.res_d, res_p=self.res_p, mu=mu)
            nd, npr, cmax, cmu = (float(v) for v in self.red[0, :4].cpu())
            nr = max(nd, npr)
            e0 = max(nr, cmax)
            if e0 <= o["tol"]:
                status = "Optimal"
                break
            if it == o["max_iter"]:
                break
            if max(nr, cmu) <= o["kappa_eps"] * mu and mu > o["tol"] / 10.0:
                # barrier update, filter reset; the right-hand side and the
                # complementarity error depend on mu: recompute them at the new mu and repeat
                # the update while the error is already below kappa_eps mu
                while True:
                    mu = max(o["tol"] / 10.0, min(o["kappa_mu"] * mu, mu ** o["theta_mu"]))
                    filt = []
                    ipm_rhs(n, m_E, m_I, self.Kxy, self.c, self.g_E, self.P, self.lo, self.up, self.zl, self.zu,
                            self.y, mu, self.sigma, self.r, self.q, self.res_d, self.res_p)
                    ipm_reduce(0, n, m_E, m_I, self.red[0], self.rwork, self.P, self.lo, self.up, zl=self.zl,
                               zu=self.zu, res_d=self.res_d, res_p=self.res_p, mu=mu)
                    cmu = float(self.red[0, 3].cpu())
                    if max(nr, cmu) > o["kappa_eps"] * mu or mu <= o["tol"] / 10.0:
                        break
            # ---- the hot path: condense + factor (inertia-corrected) + solve
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            ic = self.ic.solve(mu)
            t1.record()
            dirn = self.step.dirn
            ipm_directions(n, m_E, m_I, dirn, self.q, self.sigma, self.P, self.lo, self.up, self.zl, self.zu, mu,
                           self.dP, self.dzl, self.dzu, self.dx0)
            tau = max(o["tau_min"], 1.0 - mu)
            step_vectors(n + m_I, self.P, self.dP, self.lo, self.up, self.zl, self.zu, self.dzl, self.dzu, tau, mu,
                         self.vout, None, self.vstatus, self.vwork)
            self._k0(self.dx0, self.Kd)
            ipm_reduce(1, n, m_E, m_I, self.red[1], self.rwork, self.P, self.lo, self.up, dP=self.dP, y=self.y,
                       c=self.c, Kxy=self.Kxy, Kd=self.Kd, res_p=self.res_p, mu=mu)
            vals = self.red[1, :6].cpu().numpy()
            vo = self.vout[:2].cpu().numpy()
            st = int(self.vstatus.item())
            if st != 0:
                raise_for(st, "IPM step vectors")
            newton_ms.append(t0.elapsed_time(t1))
            a_max, a_d = float(vo[0]), float(vo[1])
            f0, gdx, dHd, gphi_b, theta0, B0 = (float(v) for v in vals)
            gphi = gdx + gphi_b
            phi0 = f0 - mu * B0
            alpha = a_max
            accepted = False
            ntrial = 0
            while alpha >= o["alpha_min_frac"] * a_max:
                ntrial += 1
                ipm_reduce(2, n, m_E, m_I, self.red[2], self.rwork, self.P, self.lo, self.up, dP=self.dP,
                           Kd=self.Kd, res_p=self.res_p, mu=mu, alpha=alpha)
                th, Ba = (float(v) for v in self.red[2, :2].cpu())
                ph = f0 + alpha * gdx + 0.5 * alpha * alpha * dHd - mu * Ba
                if all(th < tf or ph < pf for tf, pf in filt):
                    switching = gphi < 0 and alpha * (-gphi) ** o["s_phi"] > o["delta"] * theta0 ** o["s_theta"]
                    if switching:
                        if ph <= phi0 + o["eta_phi"] * alpha * gphi:
                            accepted = True
                            break
                    elif th <= (1 - o["gamma_theta"]) * theta0 or ph <= phi0 - o["gamma_phi"] * theta0:
                        filt.append(((1 - o["gamma_theta"]) * theta0, phi0 - o["gamma_phi"] * theta0))
                        accepted = True
                        break
                alpha *= 0.5
            if not accepted:
                status = "RestorationNeeded"
                break
            ipm_apply(n, m_E, m_I, self.P, self.zl, self.zu, self.y, self.xy, self.dP, self.dzl, self.dzu,
                      dirn[n:n + m] if m else self.y, self.lo, self.up, alpha, a_d, mu, o["kappa_Sigma"])
            fst = factor_stats(self.step.fwork)
            rec = dict(it=it, mu=mu, e0=e0, alpha=alpha, alpha_d=a_d, alpha_max=a_max, trials=ntrial,
                       delta_w=ic["delta_w"], inertia=ic["inertia"], theta=theta0, phi=phi0,
                       newton_ms=newton_ms[-1], panels=fst[0], swaps=fst[1], exact_cols=fst[2])
            hist.append(rec)
            if log:
                log(rec)
        torch.cuda.synchronize()
        secs = time.perf_counter() - t_start
        return dict(status=status, iterations=it, mu=mu, e0=e0, history=hist, seconds=secs, newton_ms=newton_ms)

    # -- host views --------------------------------------------------------
    def solution(self):
        n, m = self.n, self.m
        P = self.P.cpu().numpy()
        return dict(x=P[:n], s=P[n:], y=self.y[:m].cpu().numpy(), zl=self.zl[:n].cpu().numpy(),
                    zu=self.zu[:n].cpu().numpy(), vl=self.zl[n:].cpu().numpy(), vu=self.zu[n:].cpu().numpy())
