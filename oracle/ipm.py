"""CPU oracle of the interior-point loop around the hot path -- TEST INFRASTRUCTURE ONLY.

A plain primal-dual filter line-search IPM (the method of
Wachter & Biegler that HiOp implements) on the convex QP of mdsgen.QPProblem,
written out step by step in numpy, with every Newton system solved by this
package's own O1-O7 (condensation Eq.(5)->(6), Bunch-Kaufman, inertia
correction O9, solve, recovery, step vectors).  Readings (R23):
  * problem:  min 1/2 x^T H x + c^T x  s.t.  J_E x = g_E,  J_I x - s = 0,
    h_l <= s <= h_u,  lo <= x <= up   (slacks s for the inequalities, as
    HiOp's transformation);
  * Newton system = Eq.(5) with Q = H + diag(sigma_x) (+ delta_w),
    D_h = sigma_s of the slacks (reading R16), right-hand side from the
    barrier KKT residuals (derivation in DESIGN.md R23);
  * barrier update: when e_mu <= kappa_eps mu,
    mu <- max(tol/10, min(kappa_mu mu, mu^theta_mu)) and the filter is reset;
  * fraction to the boundary tau = max(tau_min, 1 - mu) (R11);
  * filter line search: backtracking alpha <- alpha/2 from
    alpha_max, filter acceptance with margins gamma_theta / gamma_phi, Armijo
    on phi under the switching condition, filter augmentation otherwise;
    theta = ||(J_E x - g_E, J_I x - s)||_1 (linear constraints: theta at a trial
    point is evaluated from r + alpha (J dx - (0, ds))), phi = f - mu sum log(gaps);
    no second-order corrections / restoration (out of scope);
  * y steps with the primal alpha, bound duals with alpha_d, then the dual
    safeguard clip with kappa_Sigma;
  * stopping: e_0 <= tol with unscaled inf-norms (s_d = s_c = 1).
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import (ERR_NOT_INTERIOR, OracleError, inertia_correction, kkt_matvec, step_vectors)

INF = 1e20
OPTS = dict(tol=1e-8, mu0=0.1, max_iter=200, tau_min=0.99, kappa_mu=0.2, theta_mu=1.5, kappa_eps=10.0,
            gamma_theta=1e-5, gamma_phi=1e-5, s_theta=1.1, s_phi=2.3, eta_phi=1e-4, delta=1.0,
            kappa_Sigma=1e10, alpha_min_frac=1e-14)


def _qp_K0(qp):
    """The Eq.(5) block structure with sigma = delta = 0 and D_y = 0: K0 (x; y) = (H x + J^T y, J x)."""
    b = qp.base
    m_I = b.m_I
    return dataclasses.replace(b, sigma_s=np.zeros(b.n_s), sigma_d=np.zeros(b.n_d), d_h=np.full(m_I, np.inf),
                               delta_w=0.0, delta_c=0.0)


def _gaps(v, lo, up):
    fl, fu = np.abs(lo) < INF, np.abs(up) < INF
    return fl, fu, np.where(fl, v - lo, 1.0), np.where(fu, up - v, 1.0)


def solve(qp, opts=None, log=None):
    """Run the IPM.  Returns dict(status, x, s, y, zl, zu, vl, vu, iterations, mu, e0, history)."""
    o = dict(OPTS, **(opts or {}))
    b = qp.base
    n_s, n_d, m_E, m_I = b.n_s, b.n_d, b.m_E, b.m_I
    n, m = n_s + n_d, m_E + m_I
    K0 = _qp_K0(qp)
    # ---- initial point: x_star (strictly interior and feasible), s = J_I x, y = 0, z = mu0 / gap
    x = np.array(qp.x_star, dtype=np.float64)
    Jx = kkt_matvec(K0, np.concatenate([x, np.zeros(m)]))[n:]
    s = Jx[m_E:].copy()
    y = np.zeros(m)
    mu = o["mu0"]
    flx, fux, glx, gux = _gaps(x, qp.lo, qp.up)
    fls, fus, gls, gus = _gaps(s, qp.h_l, qp.h_u)
    if (glx[flx] <= 0).any() or (gux[fux] <= 0).any() or (gls[fls] <= 0).any() or (gus[fus] <= 0).any():
        raise OracleError(ERR_NOT_INTERIOR, "initial point not interior")
    zl = np.where(flx, mu / glx, 0.0)
    zu = np.where(fux, mu / gux, 0.0)
    vl = np.where(fls, mu / gls, 0.0)
    vu = np.where(fus, mu / gus, 0.0)
    filt = []
    dw_last = 0.0
    hist = []
    status = "MaxIter"
    it = 0
    for it in range(o["max_iter"] + 1):
        flx, fux, glx, gux = _gaps(x, qp.lo, qp.up)
        fls, fus, gls, gus = _gaps(s, qp.h_l, qp.h_u)
        Kxy = kkt_matvec(K0, np.concatenate([x, y]))          # (H x + J^T y, J x)
        r_d = Kxy[:n] + qp.c - zl + zu                         # stationarity in x
        r_s = -y[m_E:] - vl + vu                               # stationarity in s
        r_p = Kxy[n:] - np.concatenate([qp.g_E, s])            # (J_E x - g_E, J_I x - s)
        cl, cu = np.where(flx, glx * zl, 0.0), np.where(fux, gux * zu, 0.0)
        sl, su = np.where(fls, gls * vl, 0.0), np.where(fus, gus * vu, 0.0)
        comp = np.concatenate([cl[flx], cu[fux], sl[fls], su[fus]])
        nr = max(np.abs(r_d).max(initial=0.0), np.abs(r_s).max(initial=0.0), np.abs(r_p).max(initial=0.0))
        e0 = max(nr, np.abs(comp).max(initial=0.0))
        if e0 <= o["tol"]:
            status = "Optimal"
            break
        if it == o["max_iter"]:
            break
        # barrier update (possibly several times at one point), filter reset
        while True:
            emu = max(nr, np.abs(comp - mu).max(initial=0.0))
            if emu > o["kappa_eps"] * mu or mu <= o["tol"] / 10.0:
                break
            mu = max(o["tol"] / 10.0, min(o["kappa_mu"] * mu, mu ** o["theta_mu"]))
            filt = []
        # ---- Newton system, Eq.(5): Q = H + diag(sigma_x), D_h = sigma of the slacks
        sig_x = np.where(flx, zl / glx, 0.0) + np.where(fux, zu / gux, 0.0)
        d_h = np.where(fls, vl / gls, 0.0) + np.where(fus, vu / gus, 0.0)
        bx = np.where(flx, mu / glx, 0.0) - np.where(fux, mu / gux, 0.0)
        r_x = -(Kxy[:n] + qp.c - bx)
        q = y[m_E:] + np.where(fls, mu / gls, 0.0) - np.where(fus, mu / gus, 0.0)
        r_y = np.concatenate([-r_p[:m_E], -r_p[m_E:] + q / d_h])
        prob = dataclasses.replace(b, sigma_s=sig_x[:n_s], sigma_d=sig_x[n_s:], d_h=d_h, delta_w=0.0, delta_c=0.0,
                                   r=np.concatenate([r_x, r_y]))
        ic = inertia_correction(prob, mu, delta_w_last=dw_last)
        dw_last = ic["delta_w_last"]
        dx = np.concatenate([ic["dx_s"], ic["dxy"][:n_d]])
        dy = ic["dxy"][n_d:]
        ds = (dy[m_E:] + q) / d_h
        dzl = np.where(flx, mu / glx - zl - (zl / glx) * dx, 0.0)
        dzu = np.where(fux, mu / gux - zu + (zu / gux) * dx, 0.0)
        dvl = np.where(fls, mu / gls - vl - (vl / gls) * ds, 0.0)
        dvu = np.where(fus, mu / gus - vu + (vu / gus) * ds, 0.0)
        # ---- step to the boundary over (x, s) / (z, v): O7 on the stacked vectors
        tau = max(o["tau_min"], 1.0 - mu)
        P = np.concatenate([x, s])
        st, sv, _ = step_vectors(P, np.concatenate([dx, ds]), np.concatenate([qp.lo, qp.h_l]),
                                 np.concatenate([qp.up, qp.h_u]), np.concatenate([zl, vl]), np.concatenate([zu, vu]),
                                 np.concatenate([dzl, dvl]), np.concatenate([dzu, dvu]), tau, mu, want_sigma=False)
        if st != 0:
            raise OracleError(st, "step vectors")
        a_max, a_d = sv["alpha_p"], sv["alpha_d"]
        # ---- filter line search on (theta, phi)
        Kd = kkt_matvec(K0, np.concatenate([dx, np.zeros(m)]))   # (H dx, J dx)
        dr_p = Kd[n:] - np.concatenate([np.zeros(m_E), ds])
        Hx = Kxy[:n] - kkt_matvec(K0, np.concatenate([np.zeros(n), y]))[:n]
        f0 = 0.5 * x @ Hx + qp.c @ x
        gdx = (Hx + qp.c) @ dx
        dHd = dx @ Kd[:n]
        gphi = gdx - bx @ dx + (-np.where(fls, mu / gls, 0.0) + np.where(fus, mu / gus, 0.0)) @ ds

        def barrier(al):
            xa, sa = x + al * dx, s + al * ds
            _, _, l1, u1 = _gaps(xa, qp.lo, qp.up)
            _, _, l2, u2 = _gaps(sa, qp.h_l, qp.h_u)
            return (np.log(l1[flx]).sum() + np.log(u1[fux]).sum() + np.log(l2[fls]).sum() + np.log(u2[fus]).sum())

        theta0 = np.abs(r_p).sum()
        phi0 = f0 - mu * barrier(0.0)
        alpha = a_max
        accepted = False
        ntrial = 0
        while alpha >= o["alpha_min_frac"] * a_max:
            ntrial += 1
            th = np.abs(r_p + alpha * dr_p).sum()
            ph = f0 + alpha * gdx + 0.5 * alpha * alpha * dHd - mu * barrier(alpha)
            ok_filter = all(th < tf or ph < pf for tf, pf in filt)
            if ok_filter:
                switching = gphi < 0 and alpha * (-gphi) ** o["s_phi"] > o["delta"] * theta0 ** o["s_theta"]
                if switching:
                    armijo = ph <= phi0 + o["eta_phi"] * alpha * gphi
                    if armijo:
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
        # ---- accept: primal + y with alpha, bound duals with alpha_d, dual safeguard
        x = x + alpha * dx
        s = s + alpha * ds
        y = y + alpha * dy
        zl, zu, vl, vu = zl + a_d * dzl, zu + a_d * dzu, vl + a_d * dvl, vu + a_d * dvu
        flx, fux, glx, gux = _gaps(x, qp.lo, qp.up)
        fls, fus, gls, gus = _gaps(s, qp.h_l, qp.h_u)
        kS = o["kappa_Sigma"]
        zl = np.where(flx, np.clip(zl, mu / (kS * glx), kS * mu / glx), 0.0)
        zu = np.where(fux, np.clip(zu, mu / (kS * gux), kS * mu / gux), 0.0)
        vl = np.where(fls, np.clip(vl, mu / (kS * gls), kS * mu / gls), 0.0)
        vu = np.where(fus, np.clip(vu, mu / (kS * gus), kS * mu / gus), 0.0)
        rec = dict(it=it, mu=mu, e0=e0, alpha=alpha, alpha_d=a_d, alpha_max=a_max, trials=ntrial,
                   delta_w=ic["delta_w"], inertia=ic["inertia"], theta=theta0, phi=phi0)
        hist.append(rec)
        if log:
            log(rec)
    return dict(status=status, x=x, s=s, y=y, zl=zl, zu=zu, vl=vl, vu=vu, iterations=it, mu=mu, e0=e0,
                history=hist)
