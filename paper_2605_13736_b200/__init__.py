"""paper_2605_13736_b200 — B200-native condensed-KKT hot path of the MDS IPM.

Thin Python binding (argument marshalling only) over the C-ABI library
``libmds_b200.so`` declared in ``include/mds.h``:  ``mds_condense``,
``mds_factor``, ``mds_solve``, ``ipm_step_vectors`` (§2, Eq.(5)-(6),
K1-K4 of PAPER.md:182-191).  Every step of the path runs in the library's
sm_100a kernels; PyTorch provides device memory, streams and process groups.

There is NO CPU fallback: importing this package on a box without the built
library raises, and every call requires CUDA tensors.
"""
from __future__ import annotations

import ctypes
import os

import torch

from .errors import (MDSError, DimensionError, MalformedMatrixError, CompressionError, NumericError,
                     SingularError, NotInteriorError, CudaError, WorkspaceError, raise_for)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmds_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"paper_2605_13736_b200: native library {LIB_PATH} is missing — run "
                      "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")

_lib = ctypes.CDLL(LIB_PATH)
_P, _I64, _D, _I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int32
_lib.mds_version.restype = ctypes.c_char_p
_lib.mds_plan_create.argtypes = [_I64, _I64, _I64, _I64, _P, _P, ctypes.POINTER(ctypes.c_void_p)]
_lib.mds_plan_destroy.argtypes = [_P]
_lib.mds_plan_dims.argtypes = [_P, _P]
_lib.mds_condense.argtypes = [_P, _P, _P, _P, _P, _I64, _P, _P, _I64, _P, _D, _D, _P, _P, _I64, _P, _P, _P, _P, _P,
                              ctypes.c_size_t, _P]
_lib.mds_condense_workspace_size.restype = ctypes.c_size_t
_lib.mds_condense_workspace_size.argtypes = [_P, _I64]
_lib.mds_condense_batched.argtypes = ([_P, _I64] + [_P, _I64] * 3 + [_P, _I64, _I64] + [_P, _I64] + [_P, _I64, _I64] +
                                      [_P, _I64] + [_P, _P] + [_P, _I64] + [_P, _I64, _I64] + [_P, _I64] * 2 +
                                      [_P, _P, _P, _P, ctypes.c_size_t, _P])
_lib.mds_condense_batched.restype = ctypes.c_int
_lib.mds_factor_tol.argtypes = [_P, _P, _P]
_lib.mds_factor_tol.restype = ctypes.c_int
_lib.mds_factor_workspace_size.restype = ctypes.c_size_t
_lib.mds_factor_workspace_size.argtypes = [_I64]
_lib.mds_factor.argtypes = [_I64, _P, _I64, _P, _D, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]
_lib.mds_solve_workspace_size.restype = ctypes.c_size_t
_lib.mds_solve_workspace_size.argtypes = [_I64]
_lib.mds_solve.argtypes = [_P, _I64, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _D, _P, _P, _P, ctypes.c_size_t, _P]
_lib.ipm_step_vectors_workspace_size.restype = ctypes.c_size_t
_lib.ipm_step_vectors_workspace_size.argtypes = [_I64]
_lib.ipm_step_vectors.argtypes = [_I64, _P, _P, _P, _P, _P, _P, _P, _P, _D, _D, _I32, _P, _P, _P, _P, _P, _P,
                                  ctypes.c_size_t, _P]
_lib.mds_launch_count.restype = ctypes.c_ulonglong
_lib.mds_profile_begin.restype = ctypes.c_int
_lib.mds_profile_end.restype = ctypes.c_int
_lib.mds_profile_end.argtypes = [_P, _P, ctypes.c_int]
_lib.mds_factor_panels.restype = ctypes.c_int64
_lib.mds_factor_panels.argtypes = [_P, _I64, _P, _I64]
for _f in ("mds_plan_create", "mds_plan_destroy", "mds_plan_dims", "mds_condense", "mds_factor", "mds_solve",
           "ipm_step_vectors"):
    getattr(_lib, _f).restype = ctypes.c_int

_lib.mds_factor_batched_workspace_size.restype = ctypes.c_size_t
_lib.mds_factor_batched_workspace_size.argtypes = [_I64, _I64]
_lib.mds_factor_batched.argtypes = [_I64, _I64, _P, _I64, _I64, _P, _I64, _D, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]
_lib.mds_factor_batched.restype = ctypes.c_int
_lib.mds_solve_batched_workspace_size.restype = ctypes.c_size_t
_lib.mds_solve_batched_workspace_size.argtypes = [_I64, _I64]
_lib.mds_solve_batched.argtypes = ([_P, _I64, _I64, _P, _I64, _I64] + [_P, _I64] * 7 + [_D, _P, _P, _P, ctypes.c_size_t, _P])
_lib.mds_solve_batched.restype = ctypes.c_int
_lib.ipm_step_vectors_batched_workspace_size.restype = ctypes.c_size_t
_lib.ipm_step_vectors_batched_workspace_size.argtypes = [_I64, _I64]
_lib.ipm_step_vectors_batched.argtypes = ([_I64, _I64, _I64] + [_P] * 8 + [_D, _D, _P, _P, ctypes.c_int32, _P, _P, _P,
                                          _P, _I64, _P, _P, _P, ctypes.c_size_t, _P])
_lib.ipm_step_vectors_batched.restype = ctypes.c_int

_lib.ipm_workspace_size.restype = ctypes.c_size_t
_lib.ipm_workspace_size.argtypes = [_I64, _I64]
_lib.ipm_rhs.argtypes = [_I64, _I64, _I64] + [_P] * 9 + [_D] + [_P] * 5 + [_P]
_lib.ipm_directions.argtypes = [_I64, _I64, _I64] + [_P] * 8 + [_D] + [_P] * 4 + [_P]
_lib.ipm_reduce.argtypes = [ctypes.c_int, _I64, _I64, _I64] + [_P] * 12 + [_D, _D, _P, _P, ctypes.c_size_t, _P]
_lib.ipm_apply.argtypes = [_I64, _I64, _I64] + [_P] * 11 + [_D, _D, _D, _D, _P]
for _f in ("ipm_rhs", "ipm_directions", "ipm_reduce", "ipm_apply"):
    getattr(_lib, _f).restype = ctypes.c_int

_lib.mds_kkt_residual_workspace_size.restype = ctypes.c_size_t
_lib.mds_kkt_residual_workspace_size.argtypes = [ctypes.c_void_p]
_lib.mds_kkt_residual.argtypes = [_P, _P, _P, _P, _P, _I64, _P, _P, _I64, _P, _D, _D, _P, _P, _P, _P, _P,
                                  ctypes.c_size_t, _P]
_lib.mds_kkt_residual.restype = ctypes.c_int

EXPORTS = ["mds_condense_workspace_size", "mds_condense_batched", "mds_factor_tol", "mds_kkt_residual_workspace_size", "mds_kkt_residual", "mds_version", "mds_plan_create", "mds_plan_destroy", "mds_plan_dims", "mds_condense",
           "mds_factor_workspace_size", "mds_factor", "mds_solve_workspace_size", "mds_solve",
           "ipm_step_vectors_workspace_size", "ipm_step_vectors", "mds_launch_count", "mds_profile_begin",
           "mds_profile_end", "mds_factor_panels", "mds_factor_set_grid_cap", "mds_profile_timeline", "mds_set_variant",
           "mds_factor_batched_workspace_size", "mds_factor_batched", "mds_solve_batched_workspace_size",
           "mds_solve_batched", "ipm_step_vectors_batched_workspace_size", "ipm_step_vectors_batched",
           "ipm_workspace_size", "ipm_rhs", "ipm_directions", "ipm_reduce", "ipm_apply", "mds_factor_stats",
           "mds_ic_begin_batched", "mds_ic_step_batched", "mds_ic_graph_create", "mds_ic_graph_launch",
           "mds_ic_graph_destroy", "mds_dist_panel", "mds_dist_update", "mds_dist_trsv64", "mds_dist_gemv_n",
           "mds_dist_gemv_t", "mds_dist_rowabs"]

PROF_CLASSES = ["condense_rows", "condense_norm", "condense_tiles", "anorm", "panel_diag", "panel_trsm", "panel_store",
                "panel_exact", "update", "finalize", "solve_gather", "solve_fwd", "solve_d", "solve_bwd",
                "solve_scatter", "recover", "vectors", "condense_diag", "condense_dense"]


def version() -> str:
    return _lib.mds_version().decode()


class DevPtr:
    """A raw device address inside a live CUDA tensor (a strided per-scenario view
    of a [B, W] tensor passed by its base address; the stride is a separate
    argument of the batched calls).  Keeps the tensor alive."""

    def __init__(self, t: torch.Tensor, offset_elems: int = 0):
        if not t.is_cuda:
            raise DimensionError("tensor must live on a CUDA device (no CPU fallback)")
        self.t = t
        self.ptr = t.data_ptr() + int(offset_elems) * t.element_size()
        self.dtype = t.dtype


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, DevPtr):
        return t.ptr
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch tensor")
    if not t.is_cuda:
        raise DimensionError("tensor must live on a CUDA device (no CPU fallback)")
    if not t.is_contiguous():
        raise DimensionError("tensor must be contiguous")
    return t.data_ptr()


def _f64(t, n=None):
    if isinstance(t, DevPtr):
        if t.dtype != torch.float64:
            raise DimensionError("FP64 tensor required")
        return t.ptr
    if t is not None and t.dtype != torch.float64:
        raise DimensionError("FP64 tensor required")
    if t is not None and n is not None and t.numel() < n:
        raise DimensionError(f"tensor has {t.numel()} elements, need {n}")
    return _ptr(t)


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _check(code, what):
    if code != 0:
        raise_for(code, what)


class Plan:
    """mds_plan: the J_s sparsity pattern (host CSR, rows = sparse variables),
    validated and uploaded once; fixed across IPM iterations."""

    def __init__(self, n_s, n_d, m_E, m_I, rowptr, colidx):
        import numpy as np
        rp = np.ascontiguousarray(np.asarray(rowptr), dtype=np.int32)
        ci = np.ascontiguousarray(np.asarray(colidx), dtype=np.int32)
        if rp.shape[0] != n_s + 1:
            raise DimensionError("rowptr must have n_s+1 entries")
        h = ctypes.c_void_p()
        code = _lib.mds_plan_create(n_s, n_d, m_E, m_I, rp.ctypes.data if n_s >= 0 else None,
                                    ci.ctypes.data if ci.size else None, ctypes.byref(h))
        _check(code, "mds_plan_create")
        self._h = h
        self.n_s, self.n_d, self.m_E, self.m_I = int(n_s), int(n_d), int(m_E), int(m_I)
        self.nnz = int(rp[-1]) if n_s > 0 else 0

    @property
    def handle(self):
        return self._h

    @property
    def N(self):
        return self.n_d + self.m_E + self.m_I

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.mds_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def condense_workspace_size(plan: Plan, batch: int = 1) -> int:
    return int(_lib.mds_condense_workspace_size(plan.handle, int(batch)))


def condense(plan: Plan, js_val, h_ss, sigma_s, H_dd, ldh, sigma_d, J_d, ldj, d_h, delta_w, delta_c, r,
             M, ldm, rhs_c, w_out, status, stream=None, anorm_out=None, work=None):
    """mds_condense (Eq.(5)->Eq.(6), ||M||_inf into anorm_out); see include/mds.h.
    `work`: a uint8 device tensor of condense_workspace_size(plan) bytes (allocated
    here when None -- pass one in for graph capture / no allocation per call)."""
    if work is None:
        work = torch.empty(condense_workspace_size(plan), dtype=torch.uint8, device=M.device)
    code = _lib.mds_condense(plan.handle, _f64(js_val), _f64(h_ss), _f64(sigma_s), _f64(H_dd), int(ldh),
                             _f64(sigma_d), _f64(J_d), int(ldj), _f64(d_h), float(delta_w), float(delta_c),
                             _f64(r), _f64(M), int(ldm), _f64(rhs_c), _f64(w_out), _f64(anorm_out), _ptr(status),
                             _ptr(work), work.numel() * work.element_size(), _stream(stream))
    _check(code, "mds_condense")


def condense_batched(plan: Plan, batch, js_val, h_ss, sigma_s, H_dd, ldh, sigma_d, J_d, ldj, d_h, delta_w, delta_c,
                     r, M, ldm, rhs_c, w_out, anorm_out, status, work, strides, stream=None, active=None):
    """mds_condense_batched: `strides` = dict of per-scenario element strides with keys
    val, hss, sig, H, sd, J, dh, r, M, rhs, w (every array is base + s * stride)."""
    st = strides
    code = _lib.mds_condense_batched(
        plan.handle, int(batch), _f64(js_val), int(st["val"]), _f64(h_ss), int(st["hss"]), _f64(sigma_s),
        int(st["sig"]), _f64(H_dd), int(ldh), int(st["H"]), _f64(sigma_d), int(st["sd"]), _f64(J_d), int(ldj),
        int(st["J"]), _f64(d_h), int(st["dh"]), _f64(delta_w), _f64(delta_c), _f64(r), int(st["r"]), _f64(M),
        int(ldm), int(st["M"]), _f64(rhs_c), int(st["rhs"]), _f64(w_out), int(st["w"]), _f64(anorm_out),
        _ptr(status), _ptr(active), _ptr(work), work.numel() * work.element_size(), _stream(stream))
    _check(code, "mds_condense_batched")


def factor_workspace_size(N):
    return int(_lib.mds_factor_workspace_size(int(N)))


def solve_workspace_size(N):
    return int(_lib.mds_solve_workspace_size(int(N)))


def step_vectors_workspace_size(n):
    return int(_lib.ipm_step_vectors_workspace_size(int(n)))


class Inertia(ctypes.Structure):
    _fields_ = [("pos", ctypes.c_int64), ("zero", ctypes.c_int64), ("neg", ctypes.c_int64)]


def factor(N, M, ldm, piv, zero_tol, inertia_dev, status, work, sync=True, stream=None, anorm=None):
    """mds_factor (Bunch-Kaufman LDL^T + inertia).  `anorm`: optional device scalar
    ||M||_inf from condense (else M is scanned).  Returns the inertia tuple when
    sync=True (one 24-byte D2H copy), else None."""
    host = Inertia() if sync else None
    code = _lib.mds_factor(int(N), _f64(M), int(ldm), _ptr(piv), float(zero_tol), _f64(anorm), _ptr(inertia_dev),
                           ctypes.byref(host) if sync else None, _ptr(status), _ptr(work),
                           work.numel() * work.element_size(), _stream(stream))
    _check(code, "mds_factor")
    return (host.pos, host.zero, host.neg) if sync else None


def factor_batched_workspace_size(N, batch):
    return int(_lib.mds_factor_batched_workspace_size(int(N), int(batch)))


def solve_batched_workspace_size(N, batch):
    return int(_lib.mds_solve_batched_workspace_size(int(N), int(batch)))


def step_vectors_batched_workspace_size(n, batch):
    return int(_lib.ipm_step_vectors_batched_workspace_size(int(n), int(batch)))


def factor_batched(batch, N, M, ldm, str_M, piv, str_piv, zero_tol, inertia_dev, status, work, anorm=None,
                   stream=None, active=None):
    """mds_factor_batched: `batch` factorizations in one launch sequence (never syncs).
    inertia_dev: int64 [batch, 3]; status: int32 [batch]; anorm: FP64 [batch] or None."""
    code = _lib.mds_factor_batched(int(batch), int(N), _f64(M), int(ldm), int(str_M), _ptr(piv), int(str_piv),
                                   float(zero_tol), _f64(anorm), _ptr(inertia_dev), _ptr(status), _ptr(active),
                                   _ptr(work), work.numel() * work.element_size(), _stream(stream))
    _check(code, "mds_factor_batched")


def solve_batched(plan, batch, N, LD, ldm, str_LD, piv, str_piv, rhs_c, str_rhs, js_val, str_val, w, str_w, r_xs,
                  str_r, dxy, str_dxy, dx_s, str_dxs, zero_tol, fwork, status, work, stream=None):
    """mds_solve_batched (strides in elements; see include/mds.h)."""
    code = _lib.mds_solve_batched(plan.handle if plan is not None else None, int(batch), int(N), _f64(LD), int(ldm),
                                  int(str_LD), _ptr(piv), int(str_piv), _f64(rhs_c), int(str_rhs), _f64(js_val),
                                  int(str_val), _f64(w), int(str_w), _f64(r_xs), int(str_r), _f64(dxy), int(str_dxy),
                                  _f64(dx_s), int(str_dxs), float(zero_tol), _ptr(fwork), _ptr(status), _ptr(work),
                                  work.numel() * work.element_size(), _stream(stream))
    _check(code, "mds_solve_batched")


def step_vectors_batched(batch, n, str_vec, x, dx, lo, up, zl, zu, dzl, dzu, tau, mu, out, str_out, sigma_out,
                         status, work, tau_arr=None, mu_arr=None, res=(), res_str=(), stream=None):
    """ipm_step_vectors_batched (per-scenario vectors at + s * str_vec)."""
    nres = len(res)
    arr_p = (ctypes.c_void_p * max(nres, 1))(*[_f64(t) for t in res]) if nres else None
    arr_l = (ctypes.c_int64 * max(nres, 1))(*[int(L) for L, _ in res_str]) if nres else None
    arr_s = (ctypes.c_int64 * max(nres, 1))(*[int(S) for _, S in res_str]) if nres else None
    code = _lib.ipm_step_vectors_batched(int(batch), int(n), int(str_vec), _f64(x), _f64(dx), _f64(lo), _f64(up),
                                         _f64(zl), _f64(zu), _f64(dzl), _f64(dzu), float(tau), float(mu),
                                         _f64(tau_arr), _f64(mu_arr), nres, arr_p, arr_l, arr_s, _f64(out),
                                         int(str_out), _f64(sigma_out), _ptr(status), _ptr(work),
                                         work.numel() * work.element_size(), _stream(stream))
    _check(code, "ipm_step_vectors_batched")


def factor_stats(fwork):
    """(panels, interchanges, exact-path columns, aborted) of the last mds_factor on `fwork` (synchronous)."""
    import numpy as np
    out = np.zeros(4, dtype=np.int64)
    _lib.mds_factor_stats.argtypes = [_P, _P]
    _lib.mds_factor_stats.restype = ctypes.c_int
    _check(_lib.mds_factor_stats(_ptr(fwork), out.ctypes.data), "mds_factor_stats")
    return tuple(int(v) for v in out)


def factor_tol(fwork):
    """(||M||_inf, zero-pivot tolerance) the last mds_factor on `fwork` used (synchronous)."""
    a, t = ctypes.c_double(), ctypes.c_double()
    _check(_lib.mds_factor_tol(_ptr(fwork), ctypes.byref(a), ctypes.byref(t)), "mds_factor_tol")
    return a.value, t.value


def solve(plan, N, LD, ldm, piv, rhs_c, js_val, w, r_xs, dxy, dx_s, zero_tol, fwork, status, work, stream=None):
    """mds_solve (explicit-permutation LDL^T solve + dx_s recovery)."""
    code = _lib.mds_solve(plan.handle if plan is not None else None, int(N), _f64(LD), int(ldm), _ptr(piv),
                          _f64(rhs_c), _f64(js_val), _f64(w), _f64(r_xs), _f64(dxy), _f64(dx_s), float(zero_tol),
                          _ptr(fwork), _ptr(status), _ptr(work), work.numel() * work.element_size(),
                          _stream(stream))
    _check(code, "mds_solve")


def kkt_residual_workspace_size(plan):
    """Bytes of device workspace mds_kkt_residual needs for this plan's dimensions."""
    return int(_lib.mds_kkt_residual_workspace_size(plan.handle))


def kkt_residual(plan, js_val, h_ss, sigma_s, H_dd, ldh, sigma_d, J_d, ldj, d_h, delta_w, delta_c, x, b, out,
                 rnorm=None, work=None, stream=None):
    """mds_kkt_residual: out = b - K x on the full Eq.(5) matrix (K x if b is None)."""
    if work is None:
        work = torch.empty(int(kkt_residual_workspace_size(plan)), dtype=torch.uint8,
                           device=out.device)
    code = _lib.mds_kkt_residual(plan.handle, _f64(js_val), _f64(h_ss), _f64(sigma_s), _f64(H_dd), int(ldh),
                                 _f64(sigma_d), _f64(J_d), int(ldj), _f64(d_h), float(delta_w), float(delta_c),
                                 _f64(x), _f64(b), _f64(out), _f64(rnorm), _ptr(work), work.numel(), _stream(stream))
    _check(code, "mds_kkt_residual")
    return out


def step_vectors(n, x, dx, lo, up, zl, zu, dzl, dzu, tau, mu, out, sigma_out, status, work, res=(), stream=None):
    """ipm_step_vectors (fraction-to-boundary + norms, one fused pass)."""
    nres = len(res)
    arr_p = (ctypes.c_void_p * max(nres, 1))(*[_f64(t) for t in res]) if nres else None
    arr_l = (ctypes.c_int64 * max(nres, 1))(*[t.numel() for t in res]) if nres else None
    code = _lib.ipm_step_vectors(int(n), _f64(x), _f64(dx), _f64(lo), _f64(up), _f64(zl), _f64(zu), _f64(dzl),
                                 _f64(dzu), float(tau), float(mu), nres, arr_p, arr_l, _f64(out), _f64(sigma_out),
                                 _ptr(status), _ptr(work), work.numel() * work.element_size(), _stream(stream))
    _check(code, "ipm_step_vectors")


def ipm_workspace_size(n, m_I):
    return int(_lib.ipm_workspace_size(int(n), int(m_I)))


def ipm_rhs(n, m_E, m_I, Kxy, c, g_E, P, lo, up, zl, zu, y, mu, sigma, r, q, res_d, res_p, stream=None):
    _check(_lib.ipm_rhs(int(n), int(m_E), int(m_I), _f64(Kxy), _f64(c), _f64(g_E), _f64(P), _f64(lo), _f64(up),
                        _f64(zl), _f64(zu), _f64(y), float(mu), _f64(sigma), _f64(r), _f64(q), _f64(res_d),
                        _f64(res_p), _stream(stream)), "ipm_rhs")


def ipm_directions(n, m_E, m_I, dxy, q, sigma, P, lo, up, zl, zu, mu, dP, dzl, dzu, dx0, stream=None):
    _check(_lib.ipm_directions(int(n), int(m_E), int(m_I), _f64(dxy), _f64(q), _f64(sigma), _f64(P), _f64(lo),
                               _f64(up), _f64(zl), _f64(zu), float(mu), _f64(dP), _f64(dzl), _f64(dzu), _f64(dx0),
                               _stream(stream)), "ipm_directions")


def ipm_reduce(mode, n, m_E, m_I, out, work, P, lo, up, dP=None, zl=None, zu=None, y=None, c=None, Kxy=None,
               Kd=None, res_d=None, res_p=None, mu=0.0, alpha=0.0, stream=None):
    _check(_lib.ipm_reduce(int(mode), int(n), int(m_E), int(m_I), _f64(P), _f64(dP), _f64(lo), _f64(up), _f64(zl),
                           _f64(zu), _f64(y), _f64(c), _f64(Kxy), _f64(Kd), _f64(res_d), _f64(res_p), float(mu),
                           float(alpha), _f64(out), _ptr(work), work.numel() * work.element_size(), _stream(stream)),
           "ipm_reduce")


def ipm_apply(n, m_E, m_I, P, zl, zu, y, xy, dP, dzl, dzu, dy, lo, up, alpha, alpha_d, mu, kappa_sigma,
              stream=None):
    _check(_lib.ipm_apply(int(n), int(m_E), int(m_I), _f64(P), _f64(zl), _f64(zu), _f64(y), _f64(xy), _f64(dP),
                          _f64(dzl), _f64(dzu), _f64(dy), _f64(lo), _f64(up), float(alpha), float(alpha_d),
                          float(mu), float(kappa_sigma), _stream(stream)), "ipm_apply")


class ICParamsC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("delta_w0", "delta_w_min", "delta_w_max", "kappa_w_plus",
                                              "kappa_w_plus_first", "kappa_w_minus", "delta_c_bar", "kappa_c")]


class ICStateC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("delta_w", "delta_c", "delta_w_last", "phase", "active", "ntrial",
                                              "any_active")]


class CondenseBatchedArgsC(ctypes.Structure):
    _fields_ = [("batch", _I64), ("js_val", _P), ("str_val", _I64), ("h_ss", _P), ("str_hss", _I64),
                ("sigma_s", _P), ("str_sig", _I64), ("H_dd", _P), ("ldh", _I64), ("str_H", _I64), ("sigma_d", _P),
                ("str_sd", _I64), ("J_d", _P), ("ldj", _I64), ("str_J", _I64), ("d_h", _P), ("str_dh", _I64),
                ("r", _P), ("str_r", _I64), ("M", _P), ("ldm", _I64), ("str_M", _I64), ("rhs_c", _P),
                ("str_rhs", _I64), ("w_out", _P), ("str_w", _I64), ("anorm_out", _P), ("status", _P), ("work", _P),
                ("work_bytes", ctypes.c_size_t)]


class FactorBatchedArgsC(ctypes.Structure):
    _fields_ = [("batch", _I64), ("N", _I64), ("piv", _P), ("str_piv", _I64), ("zero_tol", ctypes.c_double),
                ("inertia_dev", _P), ("work", _P), ("work_bytes", ctypes.c_size_t)]


_lib.mds_ic_begin_batched.argtypes = [_I64, _P, _P]
_lib.mds_ic_step_batched.argtypes = [_I64, _I64, _I64, _P, _P, _P, _D, _P, _P, _P]
_lib.mds_ic_graph_create.argtypes = [_P, _P, _P, _I64, _I64, _P, _D, _P, _P, ctypes.POINTER(ctypes.c_void_p)]
_lib.mds_ic_graph_launch.argtypes = [_P, _P]
_lib.mds_ic_graph_destroy.argtypes = [_P]
for _f in ("mds_ic_begin_batched", "mds_ic_step_batched", "mds_ic_graph_create", "mds_ic_graph_launch",
           "mds_ic_graph_destroy"):
    getattr(_lib, _f).restype = ctypes.c_int


def ic_begin_batched(batch, state, stream=None):
    _check(_lib.mds_ic_begin_batched(int(batch), ctypes.byref(state), _stream(stream)), "mds_ic_begin_batched")


def ic_step_batched(batch, n_d, m, inertia_dev, status, mu, params, state, mu_arr=None, stream=None):
    _check(_lib.mds_ic_step_batched(int(batch), int(n_d), int(m), _ptr(inertia_dev), _ptr(status), _f64(mu_arr),
                                    float(mu), ctypes.byref(params), ctypes.byref(state), _stream(stream)),
           "mds_ic_step_batched")


def ic_graph_create(plan, cargs, fargs, n_d, m, mu, params, state, mu_arr=None):
    h = ctypes.c_void_p()
    _check(_lib.mds_ic_graph_create(plan.handle, ctypes.byref(cargs), ctypes.byref(fargs), int(n_d), int(m),
                                    _f64(mu_arr), float(mu), ctypes.byref(params), ctypes.byref(state),
                                    ctypes.byref(h)), "mds_ic_graph_create")
    return h


def ic_graph_launch(h, stream=None):
    _check(_lib.mds_ic_graph_launch(h, _stream(stream)), "mds_ic_graph_launch")


def ic_graph_destroy(h):
    _check(_lib.mds_ic_graph_destroy(h), "mds_ic_graph_destroy")


_lib.mds_dist_panel.argtypes = [_I64, ctypes.c_int, _P, _I64, _P, _P, _I64, _P, _P, _P, _I64, _D, _P, _P, _P]
_lib.mds_dist_update.argtypes = [_I64, _I64, ctypes.c_int, _P, _P, _I64, _P, _I64, _P, _P, ctypes.c_int, _I64, _P]
_lib.mds_dist_trsv64.argtypes = [ctypes.c_int, _P, _I64, _P, ctypes.c_int, _P]
_lib.mds_dist_gemv_n.argtypes = [_I64, _I64, ctypes.c_int, _P, _I64, _P, _P, _P]
_lib.mds_dist_gemv_t.argtypes = [_I64, _I64, ctypes.c_int, _P, _I64, _P, _P, _P]
_lib.mds_dist_rowabs.argtypes = [_I64, _P, _I64, _P, _P, ctypes.c_int, _P, _P]
for _f in ("mds_dist_panel", "mds_dist_update", "mds_dist_trsv64", "mds_dist_gemv_n", "mds_dist_gemv_t",
           "mds_dist_rowabs"):
    getattr(_lib, _f).restype = ctypes.c_int


def dist_panel(n, nb, A, lda, L, W, ldl, d, cmax, parts, nparts_cap, tol, accepted, inertia, stream=None):
    _check(_lib.mds_dist_panel(int(n), int(nb), _ptr(A), int(lda), _ptr(L), _ptr(W), int(ldl), _ptr(d), _ptr(cmax),
                               _ptr(parts), int(nparts_cap), float(tol), _ptr(accepted), _ptr(inertia),
                               _stream(stream)), "mds_dist_panel")


def dist_update(N, k0, nb, L, W, ldl, C, ldc, kq, wq, nq, max_rows, stream=None):
    _check(_lib.mds_dist_update(int(N), int(k0), int(nb), _ptr(L), _ptr(W), int(ldl), _ptr(C), int(ldc), _ptr(kq),
                                _ptr(wq), int(nq), int(max_rows), _stream(stream)), "mds_dist_update")


def dist_trsv64(nb, L, ldl, y, mode, stream=None):
    _check(_lib.mds_dist_trsv64(int(nb), _ptr(L), int(ldl), _ptr(y), int(mode), _stream(stream)), "mds_dist_trsv64")


def dist_gemv_n(r0, r1, nb, L, ldl, y, acc, stream=None):
    _check(_lib.mds_dist_gemv_n(int(r0), int(r1), int(nb), _ptr(L), int(ldl), _ptr(y), _ptr(acc), _stream(stream)),
           "mds_dist_gemv_n")


def dist_gemv_t(r0, r1, nb, L, ldl, x, out, stream=None):
    _check(_lib.mds_dist_gemv_t(int(r0), int(r1), int(nb), _ptr(L), int(ldl), _ptr(x), _ptr(out), _stream(stream)),
           "mds_dist_gemv_t")


def dist_rowabs(N, C, ldc, kq, wq, nq, rs, stream=None):
    _check(_lib.mds_dist_rowabs(int(N), _ptr(C), int(ldc), _ptr(kq), _ptr(wq), int(nq), _ptr(rs), _stream(stream)),
           "mds_dist_rowabs")


def set_grid_cap(ctas: int):
    """Cap the persistent update kernels' CTAs (0 = all SMs); for concurrent streams."""
    _lib.mds_factor_set_grid_cap.argtypes = [ctypes.c_int]
    _check(_lib.mds_factor_set_grid_cap(int(ctas)), "mds_factor_set_grid_cap")


def set_variant(key: str, value: int = 1):
    """mds_set_variant: select a launch-structure variant (A/B measurement and variant
    parity tests; "default" resets all).  Results differ only by rounding order."""
    _lib.mds_set_variant.argtypes = [ctypes.c_char_p, ctypes.c_longlong]
    _lib.mds_set_variant.restype = ctypes.c_int
    _check(_lib.mds_set_variant(key.encode(), int(value)), "mds_set_variant")


def launch_count() -> int:
    """Kernels launched by the library since load (the bench's gpu_launches evidence)."""
    return int(_lib.mds_launch_count())


def profile_begin():
    _check(_lib.mds_profile_begin(), "mds_profile_begin")


def profile_end():
    """-> {class: (ms_total, launches)} for the kernels launched since profile_begin()."""
    import numpy as np
    n = len(PROF_CLASSES)
    ms = np.zeros(n)
    cnt = np.zeros(n, dtype=np.int64)
    _check(_lib.mds_profile_end(ms.ctypes.data, cnt.ctypes.data, n), "mds_profile_end")
    return {c: (float(ms[i]), int(cnt[i])) for i, c in enumerate(PROF_CLASSES)}


def profile_timeline():
    """[(class, start_ms, end_ms)] of every launch in the last profiled region."""
    import numpy as np
    _lib.mds_profile_timeline.restype = ctypes.c_int64
    _lib.mds_profile_timeline.argtypes = [_P, _I64]
    n = int(_lib.mds_profile_timeline(None, 0))
    buf = np.zeros(3 * max(n, 1))
    _lib.mds_profile_timeline(buf.ctypes.data, n)
    return [(PROF_CLASSES[int(buf[3 * i])], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n)]


def factor_panels(fwork, N):
    """Panel start columns of the last mds_factor that used `fwork` (synchronous)."""
    import numpy as np
    buf = np.zeros(N + 1, dtype=np.int32)
    n = int(_lib.mds_factor_panels(_ptr(fwork), int(N), buf.ctypes.data, N + 1))
    if n < 0:
        raise_for(n, "mds_factor_panels")
    return buf[:n].copy()


from .step import KKTStep, DeviceProblem, HostPipeline  # noqa: E402,F401
from .batch import BatchedKKTStep  # noqa: E402,F401
from .inertia import InertiaCorrection, ICParams  # noqa: E402,F401
