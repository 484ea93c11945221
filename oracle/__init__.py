"""ctypes loader for the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The product
package (paper_2603_04350_b200) never imports it; ``tests/test_abi.py`` checks that.

Every function here only marshals numpy arrays to the C oracle; the arithmetic, with
its PAPER.md citations, is in oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "oracle_cplx.c")]
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, no FFT/BLAS, -ffp-contract=off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        *(os.path.getmtime(f) for f in _SRCS), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, *_SRCS, "-lm"])
    return _LIB


class Problem(C.Structure):
    _fields_ = [
        ("dim", C.c_int),
        ("n", C.c_int),
        ("a", C.c_double),
        ("c", C.c_double),
        ("dt", C.c_double),
        ("nt", C.c_int),
        ("alpha", C.c_double),
        ("scheme", C.c_int),
        ("npoly", C.c_int),
        ("q", C.c_double * 8),
        ("a_im", C.c_double),
        ("c_im", C.c_double),
    ]


@dataclass
class Spec:
    """Problem statement u_t = (a Delta - c) u + N(u), Dirichlet on (0,1)^dim."""

    dim: int
    n: int
    a: float
    c: float
    T: float
    nt: int
    alpha: float
    scheme: int = 0  # 0 exponential Euler / ETD1, 1 ETD2
    q: tuple = field(default_factory=tuple)  # N(u) = sum_p q[p] u^p
    a_im: float = 0.0  # imaginary parts of a and c (complex state; oracle_cplx.c)
    c_im: float = 0.0

    @property
    def is_complex(self) -> bool:
        return self.a_im != 0.0 or self.c_im != 0.0

    @property
    def dt(self) -> float:
        return self.T / self.nt

    @property
    def N(self) -> int:
        return self.n ** self.dim

    def c_struct(self) -> Problem:
        p = Problem()
        p.dim, p.n, p.a, p.c, p.dt, p.nt = self.dim, self.n, self.a, self.c, self.dt, self.nt
        p.alpha, p.scheme, p.npoly = self.alpha, self.scheme, len(self.q)
        for i, v in enumerate(self.q):
            p.q[i] = v
        p.a_im, p.c_im = self.a_im, self.c_im
        return p


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        dp = C.POINTER(C.c_double)
        pp = C.POINTER(Problem)
        sig = {
            "orc_nmodes": (C.c_long, [pp]),
            "orc_axis_eigs": (None, [C.c_int, dp]),
            "orc_mode_tables": (None, [pp, dp, dp, dp, dp]),
            "orc_dst": (None, [pp, dp, dp]),
            "orc_dst_sample": (None, [pp, dp, C.POINTER(C.c_long), C.c_int, dp]),
            "orc_apply_A": (None, [pp, dp, dp]),
            "orc_nonlin": (None, [pp, dp, dp]),
            "orc_sequential": (None, [pp, dp, dp]),
            "orc_residual": (None, [pp, dp, dp, dp, dp]),
            "orc_apply_Q": (None, [pp, dp, dp]),
            "orc_apply_Qalpha": (None, [pp, dp, dp]),
            "orc_precond": (C.c_double, [pp, dp, dp]),
            "orc_fixed_point": (C.c_int, [pp, dp, dp, C.c_double, C.c_int, dp, C.POINTER(C.c_int)]),
            "orc_gmres": (C.c_int, [pp, dp, dp, C.c_double, C.c_int, C.c_int, dp, C.POINTER(C.c_int)]),
            "orc_bicgstab": (C.c_int, [pp, dp, dp, C.c_double, C.c_int, dp, C.POINTER(C.c_int)]),
            "orc_mode_residual": (None, [pp, C.c_long, dp, C.c_double, dp, dp]),
            "orc_dst_sample_batch": (None, [pp, dp, C.c_long, C.POINTER(C.c_long), C.c_int, dp]),
            "orc_dst_x_rows": (None, [pp, dp, C.c_long, dp]),
            "orc_mode_precond": (None, [pp, C.c_long, dp, dp]),
            "orc_cplx_sequential": (None, [pp, dp, dp]),
            "orc_cplx_residual": (None, [pp, dp, dp, dp, dp]),
            "orc_cplx_precond": (None, [pp, dp, dp]),
            "orc_cplx_apply_Q": (None, [pp, dp, dp]),
            "orc_cplx_fixed_point": (C.c_int, [pp, dp, dp, C.c_double, C.c_int, dp, C.POINTER(C.c_int)]),
            "orc_cplx_gmres": (C.c_int, [pp, dp, dp, C.c_double, C.c_int, C.c_int, dp, C.POINTER(C.c_int)]),
            "orc_cplx_bicgstab": (C.c_int, [pp, dp, dp, C.c_double, C.c_int, dp, C.POINTER(C.c_int)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype, f.argtypes = res, args
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def axis_eigs(n: int) -> np.ndarray:
    out = np.empty(n)
    lib().orc_axis_eigs(n, _p(out))
    return out


def mode_tables(s: Spec):
    N = s.N
    mu, E, f1, f2 = (np.empty(N) for _ in range(4))
    p = s.c_struct()
    lib().orc_mode_tables(C.byref(p), _p(mu), _p(E), _p(f1), _p(f2))
    shape = (s.n,) * s.dim
    return mu.reshape(shape), E.reshape(shape), f1.reshape(shape), f2.reshape(shape)


def dst(s: Spec, v) -> np.ndarray:
    v = _f64(v)
    out = np.empty_like(v)
    p = s.c_struct()
    lib().orc_dst(C.byref(p), _p(v), _p(out))
    return out


def dst_sample(s: Spec, v, idx) -> np.ndarray:
    v = _f64(v)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty(len(idx))
    p = s.c_struct()
    lib().orc_dst_sample(C.byref(p), _p(v), idx.ctypes.data_as(C.POINTER(C.c_long)), len(idx), _p(out))
    return out


def dst_x_rows(s: Spec, rows) -> np.ndarray:
    """The x-axis factor of V on rows [nrows][n] (the first axis pass of dst)."""
    rows = _f64(rows)
    out = np.empty_like(rows)
    p = s.c_struct()
    lib().orc_dst_x_rows(C.byref(p), _p(rows), rows.shape[0], _p(out))
    return out


def dst_sample_batch(s: Spec, V, idx) -> np.ndarray:
    """dst_sample of every slice of V [nslices][n..n] at the flat mode indices idx:
    an array [nslices][len(idx)]."""
    V = _f64(V)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    ns = V.shape[0]
    out = np.empty((ns, len(idx)))
    p = s.c_struct()
    lib().orc_dst_sample_batch(C.byref(p), _p(V), ns, idx.ctypes.data_as(C.POINTER(C.c_long)), len(idx), _p(out))
    return out


def apply_A(s: Spec, v) -> np.ndarray:
    v = _f64(v)
    out = np.empty_like(v)
    p = s.c_struct()
    lib().orc_apply_A(C.byref(p), _p(v), _p(out))
    return out


def nonlin(s: Spec, u) -> np.ndarray:
    u = _f64(u)
    out = np.empty_like(u)
    p = s.c_struct()
    lib().orc_nonlin(C.byref(p), _p(u), _p(out))
    return out


def sequential(s: Spec, u0) -> np.ndarray:
    u0 = _f64(u0)
    U = np.empty((s.nt,) + u0.shape)
    p = s.c_struct()
    lib().orc_sequential(C.byref(p), _p(u0), _p(U))
    return U


def residual(s: Spec, u0, U):
    u0, U = _f64(u0), _f64(U)
    R = np.empty_like(U)
    rn2 = C.c_double()
    p = s.c_struct()
    lib().orc_residual(C.byref(p), _p(u0), _p(U), _p(R), C.cast(C.byref(rn2), C.POINTER(C.c_double)))
    return R, rn2.value


def apply_Q(s: Spec, V) -> np.ndarray:
    V = _f64(V)
    out = np.empty_like(V)
    p = s.c_struct()
    lib().orc_apply_Q(C.byref(p), _p(V), _p(out))
    return out


def apply_Qalpha(s: Spec, V) -> np.ndarray:
    V = _f64(V)
    out = np.empty_like(V)
    p = s.c_struct()
    lib().orc_apply_Qalpha(C.byref(p), _p(V), _p(out))
    return out


def precond(s: Spec, R):
    R = _f64(R)
    S = np.empty_like(R)
    p = s.c_struct()
    leak = lib().orc_precond(C.byref(p), _p(R), _p(S))
    return S, leak


def fixed_point(s: Spec, u0, U=None, tol=1e-12, maxit=100):
    u0 = _f64(u0)
    U = np.zeros((s.nt,) + u0.shape) if U is None else _f64(U).copy()
    hist = np.zeros(maxit + 1)
    its = C.c_int()
    p = s.c_struct()
    st = lib().orc_fixed_point(C.byref(p), _p(u0), _p(U), tol, maxit, _p(hist), C.byref(its))
    return U, st, its.value, hist[: its.value + 1].copy()


def gmres(s: Spec, u0, U=None, tol=1e-12, restart=20, maxit=100):
    u0 = _f64(u0)
    U = np.zeros((s.nt,) + u0.shape) if U is None else _f64(U).copy()
    hist = np.zeros(maxit + 1)
    its = C.c_int()
    p = s.c_struct()
    st = lib().orc_gmres(C.byref(p), _p(u0), _p(U), tol, restart, maxit, _p(hist), C.byref(its))
    return U, st, its.value, hist[: its.value + 1].copy()


def bicgstab(s: Spec, u0, U=None, tol=1e-12, maxit=100):
    u0 = _f64(u0)
    U = np.zeros((s.nt,) + u0.shape) if U is None else _f64(U).copy()
    hist = np.zeros(maxit + 1)
    its = C.c_int()
    p = s.c_struct()
    st = lib().orc_bicgstab(C.byref(p), _p(u0), _p(U), tol, maxit, _p(hist), C.byref(its))
    return U, st, its.value, hist[: its.value + 1].copy()


def mode_residual(s: Spec, J: int, uhat, uhat0: float, nhat=None) -> np.ndarray:
    uhat = _f64(uhat)
    out = np.empty(s.nt)
    p = s.c_struct()
    nh_arr = _f64(nhat) if nhat is not None else None
    nh = _p(nh_arr) if nh_arr is not None else None
    lib().orc_mode_residual(C.byref(p), J, _p(uhat), float(uhat0), nh, _p(out))
    return out


def mode_precond(s: Spec, J: int, rhat) -> np.ndarray:
    rhat = _f64(rhat)
    out = np.empty(s.nt)
    p = s.c_struct()
    lib().orc_mode_precond(C.byref(p), J, _p(rhat), _p(out))
    return out


def spec(cfg) -> Spec:
    """Spec from any object with the problem fields (e.g. synth.Config)."""
    return Spec(cfg.dim, cfg.n, cfg.a, cfg.c, cfg.T, cfg.nt, cfg.alpha, cfg.scheme, tuple(cfg.q),
                getattr(cfg, "a_im", 0.0), getattr(cfg, "c_im", 0.0))


# ---- complex coefficients (oracle_cplx.c): complex128 arrays, linear problems only ----------


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def _pc(a: np.ndarray):
    assert a.dtype == np.complex128 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def cplx_sequential(s: Spec, u0) -> np.ndarray:
    u0 = _c128(u0)
    U = np.empty((s.nt,) + u0.shape, dtype=np.complex128)
    p = s.c_struct()
    lib().orc_cplx_sequential(C.byref(p), _pc(u0), _pc(U))
    return U


def cplx_residual(s: Spec, u0, U):
    u0, U = _c128(u0), _c128(U)
    R = np.empty_like(U)
    r2 = C.c_double()
    p = s.c_struct()
    lib().orc_cplx_residual(C.byref(p), _pc(u0), _pc(U), _pc(R), C.byref(r2))
    return R, r2.value


def cplx_precond(s: Spec, R) -> np.ndarray:
    R = _c128(R)
    S = np.empty_like(R)
    p = s.c_struct()
    lib().orc_cplx_precond(C.byref(p), _pc(R), _pc(S))
    return S


def cplx_apply_Q(s: Spec, V) -> np.ndarray:
    V = _c128(V)
    out = np.empty_like(V)
    p = s.c_struct()
    lib().orc_cplx_apply_Q(C.byref(p), _pc(V), _pc(out))
    return out


def cplx_fixed_point(s: Spec, u0, U=None, tol=1e-12, maxit=100):
    u0 = _c128(u0)
    U = np.zeros((s.nt,) + u0.shape, dtype=np.complex128) if U is None else _c128(U).copy()
    hist = np.zeros(maxit + 1)
    its = C.c_int()
    p = s.c_struct()
    st = lib().orc_cplx_fixed_point(C.byref(p), _pc(u0), _pc(U), tol, maxit, _p(hist), C.byref(its))
    return U, st, its.value, hist[: its.value + 1].copy()


def cplx_gmres(s: Spec, u0, U=None, tol=1e-12, restart=20, maxit=100):
    u0 = _c128(u0)
    U = np.zeros((s.nt,) + u0.shape, dtype=np.complex128) if U is None else _c128(U).copy()
    hist = np.zeros(maxit + 1)
    its = C.c_int()
    p = s.c_struct()
    st = lib().orc_cplx_gmres(C.byref(p), _pc(u0), _pc(U), tol, restart, maxit, _p(hist), C.byref(its))
    return U, st, its.value, hist[: its.value + 1].copy()


def cplx_bicgstab(s: Spec, u0, U=None, tol=1e-12, maxit=100):
    u0 = _c128(u0)
    U = np.zeros((s.nt,) + u0.shape, dtype=np.complex128) if U is None else _c128(U).copy()
    hist = np.zeros(maxit + 1)
    its = C.c_int()
    p = s.c_struct()
    st = lib().orc_cplx_bicgstab(C.byref(p), _pc(u0), _pc(U), tol, maxit, _p(hist), C.byref(its))
    return U, st, its.value, hist[: its.value + 1].copy()
