"""Inertia correction around the condensed-KKT factorization.

PAPER.md:161: the Hessian must be positive definite on the null space of the
constraint Jacobian, "checked based on the inertia of the system matrix from
(5), namely the inertia has to be (n,0,m)", and "the regularization is performed
repeatedly for increasingly large multiples until the linear solver reports that
inertia" -- adding +delta_w I to Q_{x_s}, Q_{x_d} and -delta_c I to the
constraint blocks.  Under the compression inertia(Eq.5) =
(n_s,0,0) + inertia(M), so the target for the condensed matrix is (n_d, 0, m).

The multiples follow the algorithm the paper cites for it (Wachter & Biegler
2006, "Algorithm IC"; constants as SPEC.md:354):
  IC-1  try delta_w = delta_c = 0;
  IC-2  delta_c = delta_c_bar * mu^kappa_c if the factorization showed zero
        eigenvalues, else 0;
  IC-3  delta_w = delta_w0 if delta_w_last == 0, else
        max(delta_w_min, kappa_w_minus * delta_w_last);
  IC-4  try (delta_w, delta_c); on the target inertia: delta_w_last = delta_w, done;
  IC-5  delta_w *= kappa_w_plus_first if delta_w_last == 0 else kappa_w_plus;
  IC-6  delta_w > delta_w_max -> SingularError, else back to IC-4.
(reading R22.)  delta_w enters q = h_ss + sigma_s + delta_w as well
(reading R2), so every trial re-runs mds_condense and mds_factor.

This is host control logic only: every trial's arithmetic runs in the CUDA
path (mds_condense + mds_factor); the one value that crosses the bus per trial
is the 24-byte inertia the decision needs.  The solve and step vectors run once,
for the accepted trial.
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import SingularError, raise_for


@dataclass
class ICParams:
    delta_w0: float = 1e-4
    delta_w_min: float = 1e-20
    delta_w_max: float = 1e40
    kappa_w_plus: float = 8.0
    kappa_w_plus_first: float = 100.0
    kappa_w_minus: float = 1.0 / 3.0
    delta_c_bar: float = 1e-8
    kappa_c: float = 0.25


class InertiaCorrection:
    """Inertia-corrected Newton step on one `KKTStep`.  `delta_w_last` persists
    across calls (warm start of the next Newton iteration's correction)."""

    def __init__(self, step, params: ICParams | None = None, use_graph=False):
        """use_graph: the unregularised first trial (delta_w = delta_c = 0, the usual
        accepted one) and the solve replay CUDA graphs of the step (captured on first use,
        on the caller's current stream); later trials are issued eagerly."""
        self.step = step
        self.params = params or ICParams()
        self.delta_w_last = 0.0
        self.target = (step.p.n_d, 0, step.p.m)
        self.use_graph = use_graph
        self._graphs = None

    def _attempt(self, dw, dc, trials, stream):
        self.step.p.delta_w, self.step.p.delta_c = float(dw), float(dc)
        if self.use_graph and stream is None and dw == 0.0 and dc == 0.0:
            if self._graphs is None:
                self._graphs = self.step.capture_phases()
            self._graphs[0].replay()
            ine = tuple(int(v) for v in self.step.inertia.cpu())
        else:
            ine = tuple(int(v) for v in self.step.factor_phase(stream, sync_inertia=True))
        trials.append((float(dw), float(dc), ine))
        # the stream is synchronised (inertia on the host): a data error of this trial
        # (NONPOSITIVE q_k / d_h, NONFINITE input) is final -- no delta_w escalation
        # can fix it, and its inertia is meaningless -- so raise it now
        st = int(self.step.status.item())
        if st != 0:
            raise_for(st, f"inertia correction trial (delta_w={dw:g}, delta_c={dc:g})")
        return ine

    def solve(self, mu, stream=None):
        """Factor with the smallest accepted regularisation, then solve.  Returns
        dict(delta_w, delta_c, inertia, trials=[(delta_w, delta_c, inertia), ...])."""
        P = self.params
        trials = []
        ine = self._attempt(0.0, 0.0, trials, stream)                          # IC-1
        dw = dc = 0.0
        if ine != self.target:
            dc = P.delta_c_bar * mu ** P.kappa_c if ine[1] > 0 else 0.0        # IC-2
            dw = P.delta_w0 if self.delta_w_last == 0.0 else max(P.delta_w_min,
                                                                  P.kappa_w_minus * self.delta_w_last)  # IC-3
            while True:
                ine = self._attempt(dw, dc, trials, stream)                    # IC-4
                if ine == self.target:
                    self.delta_w_last = dw
                    break
                dw *= P.kappa_w_plus_first if self.delta_w_last == 0.0 else P.kappa_w_plus   # IC-5
                if dw > P.delta_w_max:                                         # IC-6
                    raise SingularError(f"inertia correction: delta_w > {P.delta_w_max:g} "
                                        f"(last inertia {ine}, target {self.target})")
        if self._graphs is not None and stream is None and dw == 0.0 and dc == 0.0:
            self._graphs[1].replay()
        else:
            self.step.finish_phase(stream)
        return dict(delta_w=dw, delta_c=dc, inertia=ine, trials=trials)
