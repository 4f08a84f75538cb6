"""Thin ctypes binding of librexi.so (include/rexi.h) — argument marshalling only.

Every step of the REXII path runs in the library's CUDA kernels; this module only
checks tensor shapes/dtypes/devices, passes raw pointers and the current torch
stream, and turns status codes into exceptions. There is no CPU fallback: if the
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("REXI_LIB") or os.path.join(_HERE, "librexi.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built: run `python -m paper_2008_11607_b200.build` "
                      "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

REXI_OK, REXI_EINVAL, REXI_ENOMEM, REXI_ECUDA, REXI_ERANGE = range(5)
VARIANTS = {"dz": 0, "uv": 1, "dz3": 2, "pf": 3, "pfh": 4, "pfhr": 5, "pfhx": 6}
METHODS = {"rexii": 0, "rexi": 1}
SCHEDULES = {"auto": 0, "chunked": 1, "streamk": 2, "fused": 3}

_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)
_lp = ctypes.POINTER(ctypes.c_long)


class PlanInfo(ctypes.Structure):
    _fields_ = [("D", ctypes.c_int), ("variant", ctypes.c_int), ("method", ctypes.c_int),
                ("tau", ctypes.c_double),
                ("tol", ctypes.c_double), ("h", ctypes.c_double), ("mu", ctypes.c_double),
                ("M", ctypes.c_long), ("L", ctypes.c_long), ("N", ctypes.c_long),
                ("n_poles", ctypes.c_long), ("m0", ctypes.c_long), ("rho", ctypes.c_double),
                ("predicted_floor", ctypes.c_double), ("flops_per_pole_mode", ctypes.c_double),
                ("fp64_ops_per_pole_mode", ctypes.c_double), ("schedule", ctypes.c_int),
                ("last_schedule", ctypes.c_int)]


EXPORTS = {
    "rexi_plan_create": (ctypes.c_int, [ctypes.POINTER(_vp), ctypes.c_int, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_long, ctypes.c_int]),
    "rexi_plan_destroy": (ctypes.c_int, [_vp]),
    "rexi_plan_info": (ctypes.c_int, [_vp, ctypes.POINTER(PlanInfo)]),
    "rexi_plan_set_variant": (ctypes.c_int, [_vp, ctypes.c_int]),
    "rexi_plan_set_method": (ctypes.c_int, [_vp, ctypes.c_int]),
    "rexi_plan_set_graphs": (ctypes.c_int, [_vp, ctypes.c_int]),
    "rexi_plan_set_schedule": (ctypes.c_int, [_vp, ctypes.c_int]),
    "rexi_plan_set_fused_clusters": (ctypes.c_int, [_vp, ctypes.c_int]),
    "rexi_plan_set_tuning": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "rexi_plan_coeffs": (ctypes.c_int, [_vp, _dp, _dp, _dp, _dp]),
    "rexi_forward": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "rexi_poles": (ctypes.c_int, [_vp, ctypes.c_long, ctypes.c_long, _vp, _vp, _vp]),
    "rexi_poles_real": (ctypes.c_int, [_vp, ctypes.c_long, ctypes.c_long, _vp, _vp, _vp]),
    "rexi_hermitian_mirror": (ctypes.c_int, [_vp, _vp, _vp]),
    "rexi_inverse": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "rexi_apply": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rexi_apply_partial": (ctypes.c_int, [_vp, ctypes.c_long, ctypes.c_long, _vp, _vp, _vp,
                                          _vp, _vp, _vp, _vp]),
    "rexi_apply_host": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rexi_apply_host_batch": (ctypes.c_int, [_vp, ctypes.c_long, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rexi_run": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp, _vp]),
    "rexi_timing_enable": (ctypes.c_int, [_vp, ctypes.c_int]),
    "rexi_timing_read": (ctypes.c_int, [_vp, _dp, _lp, _lp]),
    "rexi_fp64_peak": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _dp, _dp]),
    "rexi_appendix_a": (ctypes.c_int, [_dp, _dp]),
    "rexi_terms_host": (ctypes.c_long, [ctypes.c_double, ctypes.c_long, ctypes.c_int, _dp, _dp, _dp, _dp]),
    "rexi_h_for_tol": (ctypes.c_double, [ctypes.c_double]),
    "rexi_fit_gaussian": (ctypes.c_int, [ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                         _dp, _dp, _dp]),
    "rexi_plan_set_table": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_double, _dp]),
    "rexi_rule_M": (ctypes.c_long, [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double]),
    "rexi_scalar_plan_create": (ctypes.c_int, [ctypes.POINTER(_vp), ctypes.c_double, ctypes.c_long,
                                               ctypes.c_int]),
    "rexi_scalar_plan_destroy": (ctypes.c_int, [_vp]),
    "rexi_scalar_plan_terms": (ctypes.c_long, [_vp]),
    "rexi_scalar_apply": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_long, _vp, _vp, _vp, ctypes.c_double,
                                         ctypes.c_double, _vp]),
    "rexi_circulant_apply": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_long, _vp, _vp, _vp, ctypes.c_double,
                                            ctypes.c_double, ctypes.c_double, _vp]),
    "rexi_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "rexi_last_error": (ctypes.c_char_p, []),
    "rexi_abi_version": (ctypes.c_int, []),
}
for _name, (_res, _args) in EXPORTS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class RexiError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = _lib.rexi_status_string(status).decode()
        detail = _lib.rexi_last_error().decode()
        super().__init__(f"{where}: {msg} ({detail})")


def _check(status, where):
    if status != REXI_OK:
        raise RexiError(status, where)


def _np_ptr(a):
    return a.ctypes.data_as(_dp)


# ----------------------------------------------------------------------------- host-only
def appendix_a():
    """(mu, a[25] complex) compiled into the library."""
    mu = ctypes.c_double()
    L = _lib.rexi_appendix_a(ctypes.byref(mu), None)
    a = np.zeros(2 * (L + 1))
    _lib.rexi_appendix_a(ctypes.byref(mu), _np_ptr(a))
    return mu.value, a[0::2] + 1j * a[1::2]


def terms_host(h, M, method="rexii"):
    """The planner's half-sum table (alpha, C1, C2, gamma) for (h, M), computed on the host.
    For method "rexi", C1 holds beta^Re_n and C2 is zero."""
    m = METHODS[method] if isinstance(method, str) else int(method)
    n = _lib.rexi_terms_host(float(h), int(M), m, None, None, None, None)
    if n < 0:
        raise ValueError("invalid h, M or method")
    al, c1, c2 = (np.zeros(2 * n) for _ in range(3))
    g = np.zeros(n)
    _lib.rexi_terms_host(float(h), int(M), m, _np_ptr(al), _np_ptr(c1), _np_ptr(c2), _np_ptr(g))
    z = lambda x: x[0::2] + 1j * x[1::2]
    return z(al), z(c1), z(c2), g


def rule_M(D, tau, tol, h=0.5):
    return int(_lib.rexi_rule_M(int(D), float(tau), float(tol), float(h)))


H_AUTO = -1.0


def h_for_tol(tol):
    return float(_lib.rexi_h_for_tol(float(tol)))


def fit_gaussian(L=24, mu=-5.133333333333333, K=200, xmax=100.0):
    """NEXT-2 refit (rexi_fit_gaussian): returns (mu, a[0..L] complex, defect); mu=None scans."""
    a = np.zeros(2 * (L + 1))
    mu_out = ctypes.c_double()
    d = ctypes.c_double()
    r = _lib.rexi_fit_gaussian(int(L), float("nan") if mu is None else float(mu), int(K), float(xmax),
                               _np_ptr(a), ctypes.byref(mu_out), ctypes.byref(d))
    if r != 0:
        raise ValueError("bad fit arguments")
    return mu_out.value, a[0::2] + 1j * a[1::2], d.value


def fp64_peak(device=0, reps=5):
    """Measured fp64-pipe rate of `device` (rexi_fp64_peak): (ops/s, best launch ms)."""
    ops = ctypes.c_double()
    ms = ctypes.c_double()
    _check(_lib.rexi_fp64_peak(int(device), int(reps), ctypes.byref(ops), ctypes.byref(ms)),
           "rexi_fp64_peak")
    return ops.value, ms.value


def abi_version():
    return _lib.rexi_abi_version()


# ----------------------------------------------------------------------------- plans
def _torch():
    import torch
    return torch


class Plan:
    """One REXII step e^{tau A} on a D x D grid (rexi_plan_create)."""

    def __init__(self, D, tau, tol=1e-12, h=0.5, M=0, device=None, variant="pfhx", method="rexii"):
        """h = "auto" (or H_AUTO) selects h_for_tol(tol) (NEXT-2)."""
        if isinstance(h, str):
            if h != "auto":
                raise ValueError("h must be a number or 'auto'")
            h = H_AUTO
        torch = _torch()
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        self._h = _vp()
        _check(_lib.rexi_plan_create(ctypes.byref(self._h), int(D), float(tau),
                                     float(tol if tol is not None else 0.0),
                                     float(h), int(M), self.device), "rexi_plan_create")
        self.set_variant(variant)
        self.set_method(method)
        inf = self.info
        self.D = inf["D"]
        self.n_poles = inf["n_poles"]

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.rexi_plan_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- metadata
    @property
    def info(self):
        i = PlanInfo()
        _check(_lib.rexi_plan_info(self._h, ctypes.byref(i)), "rexi_plan_info")
        return {k: getattr(i, k) for k, _ in PlanInfo._fields_}

    def set_variant(self, variant):
        v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
        _check(_lib.rexi_plan_set_variant(self._h, v), "rexi_plan_set_variant")
        self.variant = v

    def set_schedule(self, schedule):
        """'auto' | 'chunked' | 'streamk' distribution of the R2C pole kernel (rexi_plan_set_schedule)."""
        if schedule not in SCHEDULES:
            raise ValueError(f"schedule must be one of {sorted(SCHEDULES)}")
        _check(_lib.rexi_plan_set_schedule(self._h, SCHEDULES[schedule]), "rexi_plan_set_schedule")

    def set_fused_clusters(self, clusters):
        """Clusters the fused step splits its pole range over (0: automatic; rexi_plan_set_fused_clusters)."""
        _check(_lib.rexi_plan_set_fused_clusters(self._h, int(clusters)), "rexi_plan_set_fused_clusters")

    def set_graphs(self, enable):
        _check(_lib.rexi_plan_set_graphs(self._h, int(bool(enable))), "rexi_plan_set_graphs")

    def set_table(self, mu, a):
        """Use (mu, a_0..a_L) instead of Appendix A (rexi_plan_set_table)."""
        a = np.asarray(a, dtype=np.complex128)
        buf = np.ascontiguousarray(np.stack([a.real, a.imag], axis=-1).ravel())
        _check(_lib.rexi_plan_set_table(self._h, len(a) - 1, float(mu), _np_ptr(buf)), "rexi_plan_set_table")
        self.n_poles = self.info["n_poles"]

    def set_method(self, method):
        m = METHODS[method] if isinstance(method, str) else int(method)
        _check(_lib.rexi_plan_set_method(self._h, m), "rexi_plan_set_method")
        self.method = m

    def set_tuning(self, modes_per_thread, poles_per_iter=1, min_blocks_per_sm=4):
        """Tune the pole kernel of the current variant/method (see rexi_plan_set_tuning)."""
        _check(_lib.rexi_plan_set_tuning(self._h, int(modes_per_thread), int(poles_per_iter),
                                         int(min_blocks_per_sm)), "rexi_plan_set_tuning")

    def coeffs(self):
        n = self.n_poles
        al, c1, c2 = (np.zeros(2 * n) for _ in range(3))
        g = np.zeros(n)
        _check(_lib.rexi_plan_coeffs(self._h, _np_ptr(al), _np_ptr(c1), _np_ptr(c2), _np_ptr(g)),
               "rexi_plan_coeffs")
        z = lambda x: x[0::2] + 1j * x[1::2]
        return z(al), z(c1), z(c2), g

    # -- tensor checks
    def _stream(self):
        torch = _torch()
        return _vp(torch.cuda.current_stream(self.device).cuda_stream)

    def _field(self, t, name):
        torch = _torch()
        if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda \
                or t.device.index != self.device or tuple(t.shape) != (self.D, self.D) \
                or not t.is_contiguous():
            raise ValueError(f"{name}: expected a contiguous float64 ({self.D}, {self.D}) tensor "
                             f"on cuda:{self.device}")
        return _vp(t.data_ptr())

    def _spec(self, t, name):
        torch = _torch()
        if not isinstance(t, torch.Tensor) or t.dtype != torch.complex128 or not t.is_cuda \
                or t.device.index != self.device or tuple(t.shape) != (3, self.D, self.D) \
                or not t.is_contiguous():
            raise ValueError(f"{name}: expected a contiguous complex128 (3, {self.D}, {self.D}) "
                             f"tensor on cuda:{self.device}")
        return _vp(t.data_ptr())

    def _new_fields(self):
        torch = _torch()
        return tuple(torch.empty((self.D, self.D), dtype=torch.float64, device=f"cuda:{self.device}")
                     for _ in range(3))

    def _new_spec(self):
        torch = _torch()
        return torch.empty((3, self.D, self.D), dtype=torch.complex128, device=f"cuda:{self.device}")

    # -- the path
    def forward(self, eta, u, v, fhat=None):
        fhat = self._new_spec() if fhat is None else fhat
        _check(_lib.rexi_forward(self._h, self._field(eta, "eta"), self._field(u, "u"),
                                 self._field(v, "v"), self._spec(fhat, "fhat"), self._stream()),
               "rexi_forward")
        return fhat

    def poles(self, fhat, begin=0, end=None, acc=None):
        end = self.n_poles if end is None else end
        acc = self._new_spec() if acc is None else acc
        _check(_lib.rexi_poles(self._h, int(begin), int(end), self._spec(fhat, "fhat"),
                               self._spec(acc, "acc"), self._stream()), "rexi_poles")
        return acc

    def poles_real(self, fhat, begin=0, end=None, acc=None):
        """rexi_poles_real: the Hermitian part of the pole sum for the spectrum of real fields."""
        end = self.n_poles if end is None else end
        acc = self._new_spec() if acc is None else acc
        _check(_lib.rexi_poles_real(self._h, int(begin), int(end), self._spec(fhat, "fhat"),
                                    self._spec(acc, "acc"), self._stream()), "rexi_poles_real")
        return acc

    def hermitian_mirror(self, acc):
        """rexi_hermitian_mirror: rows D/2+1 .. D-1 of a Hermitian spectrum from rows 1 .. D/2-1."""
        _check(_lib.rexi_hermitian_mirror(self._h, self._spec(acc, "acc"), self._stream()),
               "rexi_hermitian_mirror")
        return acc

    def inverse(self, acc, out=None):
        out = self._new_fields() if out is None else out
        _check(_lib.rexi_inverse(self._h, self._spec(acc, "acc"), *(self._field(o, "out") for o in out),
                                 self._stream()), "rexi_inverse")
        return out

    def apply(self, eta, u, v, out=None):
        out = self._new_fields() if out is None else out
        _check(_lib.rexi_apply(self._h, self._field(eta, "eta"), self._field(u, "u"), self._field(v, "v"),
                               *(self._field(o, "out") for o in out), self._stream()), "rexi_apply")
        return out

    def apply_partial(self, begin, end, eta, u, v, out=None):
        out = self._new_fields() if out is None else out
        _check(_lib.rexi_apply_partial(self._h, int(begin), int(end), self._field(eta, "eta"),
                                       self._field(u, "u"), self._field(v, "v"),
                                       *(self._field(o, "out") for o in out), self._stream()),
               "rexi_apply_partial")
        return out

    def apply_host(self, eta, u, v, out=None):
        """Host buffers in and out (numpy float64 arrays or CPU tensors, ideally pinned)."""
        def ptr(a, name):
            if isinstance(a, np.ndarray):
                if a.dtype != np.float64 or a.shape != (self.D, self.D) or not a.flags.c_contiguous:
                    raise ValueError(f"{name}: expected C-contiguous float64 ({self.D}, {self.D})")
                return _vp(a.ctypes.data)
            torch = _torch()
            if a.device.type != "cpu" or a.dtype != torch.float64 or tuple(a.shape) != (self.D, self.D) \
                    or not a.is_contiguous():
                raise ValueError(f"{name}: expected a contiguous float64 CPU tensor")
            return _vp(a.data_ptr())
        if out is None:
            out = tuple(np.empty((self.D, self.D)) for _ in range(3))
        _check(_lib.rexi_apply_host(self._h, ptr(eta, "eta"), ptr(u, "u"), ptr(v, "v"),
                                    *(ptr(o, "out") for o in out), self._stream()), "rexi_apply_host")
        return out

    def apply_host_batch(self, eta, u, v, out=None):
        """`batch` independent problems from host arrays of shape (batch, D, D) (numpy float64 or
        CPU tensors, ideally pinned); copies overlap the steps (rexi_apply_host_batch)."""
        def ptr(a, name):
            if isinstance(a, np.ndarray):
                if a.dtype != np.float64 or a.ndim != 3 or a.shape[1:] != (self.D, self.D) \
                        or not a.flags.c_contiguous:
                    raise ValueError(f"{name}: expected C-contiguous float64 (batch, {self.D}, {self.D})")
                return _vp(a.ctypes.data), a.shape[0]
            torch = _torch()
            if a.device.type != "cpu" or a.dtype != torch.float64 or a.dim() != 3 \
                    or tuple(a.shape[1:]) != (self.D, self.D) or not a.is_contiguous():
                raise ValueError(f"{name}: expected a contiguous float64 CPU tensor (batch, D, D)")
            return _vp(a.data_ptr()), a.shape[0]
        ins = [ptr(x, nm) for x, nm in ((eta, "eta"), (u, "u"), (v, "v"))]
        batch = ins[0][1]
        if out is None:
            out = tuple(np.empty((batch, self.D, self.D)) for _ in range(3))
        outs = [ptr(o, "out") for o in out]
        if any(b != batch for _, b in ins + outs):
            raise ValueError("all batch arrays must have the same leading dimension")
        _check(_lib.rexi_apply_host_batch(self._h, int(batch), *(x for x, _ in ins), *(o for o, _ in outs),
                                          self._stream()), "rexi_apply_host_batch")
        return out

    def run(self, steps, eta, u, v):
        """`steps` REXII steps in place (S6, T_final = steps * tau)."""
        _check(_lib.rexi_run(self._h, int(steps), self._field(eta, "eta"), self._field(u, "u"),
                             self._field(v, "v"), self._stream()), "rexi_run")
        return eta, u, v

    # -- timing of the dominant kernel
    def timing_enable(self, on=True):
        _check(_lib.rexi_timing_enable(self._h, int(bool(on))), "rexi_timing_enable")

    def timing_read(self):
        ms = ctypes.c_double()
        pl = ctypes.c_long()
        tl = ctypes.c_long()
        _check(_lib.rexi_timing_read(self._h, ctypes.byref(ms), ctypes.byref(pl), ctypes.byref(tl)),
               "rexi_timing_read")
        return ms.value, pl.value, tl.value


SCALAR_METHODS = {"rexii": 0, "rexi": 1, "rexi_m": 2}


class ScalarPlan:
    """NEXT-3: the scalar forms per eigenvalue of a diagonalised operator (rexi_scalar_apply)."""

    def __init__(self, h, M, device=None):
        torch = _torch()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self._h = _vp()
        _check(_lib.rexi_scalar_plan_create(ctypes.byref(self._h), float(h), int(M), self.device),
               "rexi_scalar_plan_create")
        self.n_terms = _lib.rexi_scalar_plan_terms(self._h)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.rexi_scalar_plan_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def apply(self, x, vec, method="rexii", phase=1.0 + 0.0j, out=None):
        """out_j = phase * r(i x_j) * vec_j for float64 x and complex128 vec (CUDA tensors)."""
        torch = _torch()
        ok = (isinstance(x, torch.Tensor) and isinstance(vec, torch.Tensor)
              and x.dtype == torch.float64 and vec.dtype == torch.complex128 and x.shape == vec.shape
              and x.is_cuda and vec.is_cuda and x.is_contiguous() and vec.is_contiguous()
              and x.device.index == self.device and vec.device.index == self.device)
        if not ok:
            raise ValueError(f"x: contiguous float64, vec: contiguous complex128, same shape, on "
                             f"cuda:{self.device}")
        if method not in SCALAR_METHODS:
            raise ValueError(f"method must be one of {sorted(SCALAR_METHODS)}")
        out = torch.empty_like(vec) if out is None else out
        if not (isinstance(out, torch.Tensor) and out.dtype == torch.complex128 and out.shape == vec.shape
                and out.is_cuda and out.device.index == self.device and out.is_contiguous()):
            raise ValueError(f"out: expected a contiguous complex128 tensor of shape {tuple(vec.shape)} "
                             f"on cuda:{self.device}")
        stream = _vp(torch.cuda.current_stream(self.device).cuda_stream)
        _check(_lib.rexi_scalar_apply(self._h, SCALAR_METHODS[method], int(x.numel()), _vp(x.data_ptr()),
                                      _vp(vec.data_ptr()), _vp(out.data_ptr()), float(complex(phase).real),
                                      float(complex(phase).imag), stream), "rexi_scalar_apply")
        return out

    def circulant_apply(self, col, f, tau, method="rexii", nu=0.0, out=None):
        """rexi_circulant_apply: e^{tau A} f for the circulant A with first column `col` (complex128
        CUDA tensors of length n on this plan's device): library DFTs + the scalar pole kernel."""
        torch = _torch()

        def chk(t, name):
            if not (isinstance(t, torch.Tensor) and t.dtype == torch.complex128 and t.dim() == 1
                    and t.is_cuda and t.device.index == self.device and t.is_contiguous()):
                raise ValueError(f"{name}: expected a contiguous 1-D complex128 tensor on cuda:{self.device}")
            return _vp(t.data_ptr())
        if method not in SCALAR_METHODS:
            raise ValueError(f"method must be one of {sorted(SCALAR_METHODS)}")
        n = int(col.numel()) if isinstance(col, torch.Tensor) else -1
        if not isinstance(f, torch.Tensor) or f.numel() != n:
            raise ValueError("col and f must have the same length")
        out = torch.empty_like(f) if out is None else out
        if out.numel() != n or out.data_ptr() in (col.data_ptr(), f.data_ptr()):
            raise ValueError("out: length n, must not alias col or f")
        nu = complex(nu)
        stream = _vp(torch.cuda.current_stream(self.device).cuda_stream)
        _check(_lib.rexi_circulant_apply(self._h, SCALAR_METHODS[method], n, chk(col, "col"), chk(f, "f"),
                                         chk(out, "out"), float(tau), nu.real, nu.imag, stream),
               "rexi_circulant_apply")
        return out
