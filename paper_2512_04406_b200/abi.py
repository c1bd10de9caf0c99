"""Thin ctypes binding of libdrsdp.so (names follow include/drsdp.h; marshalling only).

Device buffers are passed as raw pointers (``tensor.data_ptr()`` of torch CUDA tensors: torch is
used for device memory and streams only). Host buffers are numpy float64/int32 arrays.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

OK, ERR_INVALID_ARG, ERR_NOT_SYMMETRIC, ERR_SINGULAR_AAT, ERR_STATE, ERR_CUDA, ERR_OOM, \
    ERR_NOT_CONVERGED, ERR_NUMERIC = range(9)
EVAL_COSTGRAD, EVAL_HVP = 1, 2
TRACE_COLUMNS = ("iter", "eta_p", "eta_d", "eta_g", "eta_max", "primal_obj", "dual_obj", "sigma", "p",
                 "inner_iters", "cg_iters", "escape_delta", "time_s")

EXPORTED = ("drsdp_create", "drsdp_destroy", "drsdp_last_error", "drsdp_sync", "drsdp_set_problem",
            "drsdp_set_bqp", "drsdp_set_blocks", "drsdp_set_bqp_chain", "drsdp_get_block_sizes", "drsdp_get_sizes", "drsdp_export_index_map", "drsdp_default_params",
            "drsdp_set_params", "drsdp_set_initial_factor", "drsdp_solve", "drsdp_get_solution",
            "drsdp_get_trace", "drsdp_set_subproblem_matrix", "drsdp_set_subproblem_rows", "drsdp_subproblem_eval",
            "drsdp_subproblem_eval_host", "drsdp_assemble_M", "drsdp_y_update", "drsdp_dual_update",
            "drsdp_alm_eval", "drsdp_x_eigs", "drsdp_launch_count", "drsdp_profile_enable", "drsdp_profile_read")


class DrsdpError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"drsdp error {code}: {msg}")
        self.code = code


class Params(C.Structure):
    _fields_ = [("sigma0", C.c_double), ("sigma_min", C.c_double), ("sigma_max", C.c_double),
                ("gamma", C.c_double), ("tau1", C.c_double), ("tau2", C.c_double), ("tol", C.c_double),
                ("eig_neg_tol", C.c_double), ("rank_tol", C.c_double), ("eps_scale", C.c_double),
                ("eps_floor", C.c_double), ("time_limit_s", C.c_double), ("p0", C.c_int32),
                ("max_outer", C.c_int32), ("max_rtr", C.c_int32), ("max_tcg", C.c_int32),
                ("escape_max", C.c_int32), ("mode", C.c_int32), ("seed", C.c_uint64), ("rho_reg", C.c_double),
                ("stall_rtr", C.c_int32), ("eig_method", C.c_int32), ("precond_mu", C.c_double),
                ("lanczos_steps", C.c_int32), ("hold_max", C.c_int32),
                ("escape_gate", C.c_double), ("stall_factor", C.c_double), ("hold_tau", C.c_double),
                ("sigma_boost", C.c_double)]


class Info(C.Structure):
    _fields_ = [("status", C.c_int32), ("outer_iters", C.c_int32), ("p_final", C.c_int32),
                ("p_max", C.c_int32), ("rtr_iters", C.c_int64), ("tcg_iters", C.c_int64),
                ("n_costgrad", C.c_int64), ("n_hvp", C.c_int64), ("eta_p", C.c_double),
                ("eta_d", C.c_double), ("eta_g", C.c_double), ("dual_obj", C.c_double),
                ("primal_obj", C.c_double), ("seconds", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def lib_path() -> str:
    return os.path.join(_HERE, "libdrsdp.so")


def load_library():
    """Load libdrsdp.so (raises if it has not been built: there is no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        raise DrsdpError(-1, f"{path} not built (run python -m paper_2512_04406_b200.build)")
    lib = C.CDLL(path)
    vp, i32, i64, dp = C.c_void_p, C.c_int32, C.c_int64, C.c_void_p
    sig = {
        "drsdp_create": (C.c_int, [C.POINTER(vp), C.c_int, vp]),
        "drsdp_destroy": (None, [vp]),
        "drsdp_last_error": (C.c_char_p, [vp]),
        "drsdp_sync": (C.c_int, [vp]),
        "drsdp_set_problem": (C.c_int, [vp, i64, i64, dp, i64, dp, dp, dp, dp]),
        "drsdp_set_bqp": (C.c_int, [vp, i32, dp, dp]),
        "drsdp_set_blocks": (C.c_int, [vp, i32, i32, i64, dp, dp]),
        "drsdp_set_bqp_chain": (C.c_int, [vp, i32, i32, dp, dp]),
        "drsdp_get_block_sizes": (C.c_int, [vp, C.POINTER(i32), C.POINTER(i32)]),
        "drsdp_get_sizes": (C.c_int, [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]),
        "drsdp_export_index_map": (C.c_int, [vp, dp, dp, dp]),
        "drsdp_default_params": (C.c_int, [C.POINTER(Params)]),
        "drsdp_set_params": (C.c_int, [vp, C.POINTER(Params)]),
        "drsdp_set_initial_factor": (C.c_int, [vp, i32, dp]),
        "drsdp_solve": (C.c_int, [vp, C.POINTER(Info)]),
        "drsdp_get_solution": (C.c_int, [vp, dp, dp, C.POINTER(i32), dp, dp]),
        "drsdp_get_trace": (C.c_int, [vp, i32, dp, C.POINTER(i32)]),
        "drsdp_set_subproblem_matrix": (C.c_int, [vp, i64, dp, i64]),
        "drsdp_set_subproblem_rows": (C.c_int, [vp, i64, i64, i64, dp, i64]),
        "drsdp_subproblem_eval": (C.c_int, [vp, i32, i32, dp, dp, dp, dp, dp, dp]),
        "drsdp_subproblem_eval_host": (C.c_int, [vp, i32, i32, dp, dp, dp, dp, dp, dp]),
        "drsdp_assemble_M": (C.c_int, [vp, dp, dp, i64, C.c_double, dp, i64]),
        "drsdp_y_update": (C.c_int, [vp, i32, dp, dp]),
        "drsdp_dual_update": (C.c_int, [vp, i32, dp, dp, C.c_double, dp, i64, dp, dp]),
        "drsdp_alm_eval": (C.c_int, [vp, i32, i32, dp, i64, C.c_double, dp, dp, dp, dp, dp, dp]),
        "drsdp_x_eigs": (C.c_int, [vp, dp, i64, dp, i32, i32, dp, C.POINTER(C.c_double), dp, dp,
                                   C.POINTER(i32)]),
        "drsdp_launch_count": (C.c_int, [vp, C.POINTER(i64)]),
        "drsdp_profile_enable": (C.c_int, [vp, C.c_int]),
        "drsdp_profile_read": (C.c_int, [vp, i32, C.POINTER(C.c_double), C.POINTER(i64)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _LIB = lib
    return lib


def _ptr(x):
    """Raw pointer of a torch tensor / numpy array / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def _host(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the legacy default stream handle


class Context:
    """One drsdp_ctx (one CUDA stream).

    ``stream``: a cudaStream_t integer (e.g. ``torch.cuda.Stream().cuda_stream``); 0 means the
    legacy default stream (torch's default), passed as cudaStreamLegacy; None lets the library
    create its own non-blocking stream."""

    def __init__(self, device: int = 0, stream: int | None = 0):
        self.lib = load_library()
        h = C.c_void_p()
        st = None if stream is None else (CUDA_STREAM_LEGACY if stream == 0 else stream)
        rc = self.lib.drsdp_create(C.byref(h), device, st)
        if rc != OK:
            raise DrsdpError(rc, "drsdp_create failed (no usable CUDA device?)")
        self.h = h
        self._keep = []

    def close(self):
        if getattr(self, "h", None):
            self.lib.drsdp_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, allow=()):
        if rc != OK and rc not in allow:
            msg = self.lib.drsdp_last_error(self.h)
            raise DrsdpError(rc, msg.decode() if msg else "")
        return rc

    # -- problem ---------------------------------------------------------------------------
    def set_problem(self, n, m, C_mat, row, col, cons, b):
        Cm = None if C_mat is None else _host(C_mat, np.float64)
        row, col, cons = (_host(x, np.int32) for x in (row, col, cons))
        b = _host(b, np.float64)
        return self._check(self.lib.drsdp_set_problem(self.h, n, m, _ptr(Cm), row.size, _ptr(row), _ptr(col),
                                                      _ptr(cons), _ptr(b)))

    def set_bqp(self, Q, c):
        Q = _host(Q, np.float64)
        c = _host(c, np.float64)
        return self._check(self.lib.drsdp_set_bqp(self.h, Q.shape[0], _ptr(Q), _ptr(c)))

    def set_blocks(self, amaps, b):
        """Uniform multi-block problem: amaps (t, nb, nb) int32, b (m,) (drsdp_set_blocks)."""
        amaps = _host(amaps, np.int32)
        b = _host(b, np.float64)
        t, nb = amaps.shape[0], amaps.shape[1]
        return self._check(self.lib.drsdp_set_blocks(self.h, t, nb, b.size, _ptr(amaps), _ptr(b)))

    def set_bqp_chain(self, Qs, cs):
        """Clique-chain sparse BQP relaxation: Qs (t, q, q), cs (t, q) (drsdp_set_bqp_chain)."""
        Qs = _host(Qs, np.float64)
        cs = _host(cs, np.float64)
        return self._check(self.lib.drsdp_set_bqp_chain(self.h, Qs.shape[1], Qs.shape[0], _ptr(Qs), _ptr(cs)))

    def block_sizes(self):
        t, nb = C.c_int32(), C.c_int32()
        self._check(self.lib.drsdp_get_block_sizes(self.h, C.byref(t), C.byref(nb)))
        return t.value, nb.value

    def sizes(self):
        n, m, nu = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self.lib.drsdp_get_sizes(self.h, C.byref(n), C.byref(m), C.byref(nu)))
        return n.value, m.value, nu.value

    def export_index_map(self):
        n, m, nu = self.sizes()
        t, nb = self.block_sizes()
        amap = np.empty((n, nb), np.int32)  # dense: nb = n; blocks: stacked rows
        sp = np.empty(m + 1, np.int64)
        pos = np.empty(nu, np.uint32)
        self._check(self.lib.drsdp_export_index_map(self.h, _ptr(amap), _ptr(sp), _ptr(pos)))
        return amap, sp, pos

    # -- solve -----------------------------------------------------------------------------
    @staticmethod
    def default_params(**kw) -> Params:
        prm = Params()
        load_library().drsdp_default_params(C.byref(prm))
        for k, v in kw.items():
            setattr(prm, k, v)
        return prm

    def set_params(self, prm: Params | None = None, **kw):
        if prm is None:
            prm = self.default_params(**kw)
        return self._check(self.lib.drsdp_set_params(self.h, C.byref(prm)))

    def set_initial_factor(self, Y0):
        Y0 = _host(Y0, np.float64)
        return self._check(self.lib.drsdp_set_initial_factor(self.h, Y0.shape[1], _ptr(Y0)))

    def solve(self) -> dict:
        info = Info()
        rc = self.lib.drsdp_solve(self.h, C.byref(info))
        self._check(rc, allow=(ERR_NOT_CONVERGED,))
        return info.as_dict()

    def solution(self, want_X=False):
        n, m, _ = self.sizes()
        y = np.empty(m)
        z = np.empty(n)
        p = C.c_int32()
        self._check(self.lib.drsdp_get_solution(self.h, None, None, C.byref(p), None, None))
        Y = np.empty((n, p.value))
        t, nb = self.block_sizes()
        X = (np.empty((t, nb, nb)) if t else np.empty((n, n))) if want_X else None
        self._check(self.lib.drsdp_get_solution(self.h, _ptr(y), _ptr(Y), C.byref(p), _ptr(z), _ptr(X)))
        return {"y": y, "Y": Y, "z": z, "X": X, "p": p.value}

    def trace(self):
        nr = C.c_int32()
        self._check(self.lib.drsdp_get_trace(self.h, 0, None, C.byref(nr)))
        rows = np.empty((max(nr.value, 1), 13))
        self._check(self.lib.drsdp_get_trace(self.h, nr.value, _ptr(rows), C.byref(nr)))
        return [dict(zip(TRACE_COLUMNS, r)) for r in rows[: nr.value]]

    # -- subproblem evaluation -------------------------------------------------------------
    def set_subproblem_matrix(self, n, M_dev, ldm):
        self._keep = [M_dev]
        return self._check(self.lib.drsdp_set_subproblem_matrix(self.h, n, _ptr(M_dev), ldm))

    def set_subproblem_rows(self, n, row0, row1, M_rows_dev, ldm):
        """Row-block mode (row-sharded evaluation): rows [row0, row1) of the n x n matrix."""
        self._keep = [M_rows_dev]
        return self._check(self.lib.drsdp_set_subproblem_rows(self.h, n, row0, row1, _ptr(M_rows_dev), ldm))

    def subproblem_eval(self, flags, p, Y, U=None, cost=None, egrad=None, rgrad=None, hvp=None):
        return self._check(self.lib.drsdp_subproblem_eval(self.h, flags, p, _ptr(Y), _ptr(U), _ptr(cost),
                                                          _ptr(egrad), _ptr(rgrad), _ptr(hvp)))

    def subproblem_eval_host(self, flags, Y, U=None, want_egrad=False):
        Y = _host(Y, np.float64)
        n, p = Y.shape
        U = None if U is None else _host(U, np.float64)
        cost = np.empty(1)
        eg = np.empty_like(Y) if want_egrad else None
        rg = np.empty_like(Y)
        hv = np.empty_like(Y) if flags & EVAL_HVP else None
        self._check(self.lib.drsdp_subproblem_eval_host(self.h, flags, p, _ptr(Y), _ptr(U), _ptr(cost), _ptr(eg),
                                                        _ptr(rg), _ptr(hv)))
        return {"f": float(cost[0]), "E": eg, "R": rg, "H": hv}

    def alm_eval(self, flags, p, T, ldt, sigma, Y, U=None, cost=None, egrad=None, rgrad=None, hvp=None):
        return self._check(self.lib.drsdp_alm_eval(self.h, flags, p, _ptr(T), ldt, sigma, _ptr(Y), _ptr(U),
                                                   _ptr(cost), _ptr(egrad), _ptr(rgrad), _ptr(hvp)))

    def assemble_M(self, y, T, ldt, sigma, M, ldm):
        return self._check(self.lib.drsdp_assemble_M(self.h, _ptr(y), _ptr(T), ldt, sigma, _ptr(M), ldm))

    def y_update(self, p, Y, y):
        return self._check(self.lib.drsdp_y_update(self.h, p, _ptr(Y), _ptr(y)))

    def x_eigs(self, T, ldt, z, steps, nvec, V):
        """Block-Lanczos extreme eigenpairs of X = T - Diag(z) (device T, z, V): returns
        (ritz values (nvec), residual norms (nvec), largest Ritz value, basis size)."""
        ritz = np.empty(max(nvec, 1))
        resid = np.empty(max(nvec, 1))
        lmax = C.c_double()
        basis = C.c_int32()
        self._check(self.lib.drsdp_x_eigs(self.h, _ptr(T), ldt, _ptr(z), steps, nvec, ritz.ctypes.data,
                                          C.byref(lmax), _ptr(V), resid.ctypes.data, C.byref(basis)))
        return ritz[:nvec], resid[:nvec], lmax.value, basis.value

    def dual_update(self, p, Y, y, sigma, T, ldt, z, scalars):
        return self._check(self.lib.drsdp_dual_update(self.h, p, _ptr(Y), _ptr(y), sigma, _ptr(T), ldt, _ptr(z),
                                                      _ptr(scalars)))

    def sync(self):
        return self._check(self.lib.drsdp_sync(self.h))

    def launch_count(self) -> int:
        c = C.c_int64()
        self._check(self.lib.drsdp_launch_count(self.h, C.byref(c)))
        return c.value

    def profile_enable(self, on=True):
        return self._check(self.lib.drsdp_profile_enable(self.h, 1 if on else 0))

    def profile_read(self, kind=0):
        ms, cnt = C.c_double(), C.c_int64()
        self._check(self.lib.drsdp_profile_read(self.h, kind, C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value
