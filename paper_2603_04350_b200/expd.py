"""Thin ctypes binding of libexpd.so (C-ABI: include/expd.h).

Argument marshalling only: every step of the Exp-ParaDiag path runs in the library's
CUDA kernels.  torch supplies device memory (the caller-owned workspace and vectors) and
the CUDA stream.  There is no CPU fallback: if the extension is missing or no CUDA
device is visible, constructing a Plan raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EXPD_LIB", os.path.join(_HERE, "libexpd.so"))  # override: tuning A/B only

EXPD_OK = 0
STATUS = {
    0: "EXPD_OK",
    1: "EXPD_ERR_INVALID_ARG",
    2: "EXPD_ERR_UNSUPPORTED",
    3: "EXPD_ERR_CUDA",
    4: "EXPD_ERR_NCCL",
    5: "EXPD_ERR_OOM",
    6: "EXPD_ERR_BREAKDOWN",
    7: "EXPD_ERR_NOT_CONVERGED",
}

# every symbol include/expd.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "expd_plan_create",
    "expd_plan_workspace_bytes",
    "expd_plan_set_workspace",
    "expd_plan_destroy",
    "expd_plan_last_error",
    "expd_residual",
    "expd_precond_apply",
    "expd_fixed_point_solve",
    "expd_gmres_solve",
    "expd_bicgstab_solve",
    "expd_load_state",
    "expd_sweep",
    "expd_sweep_norm2",
    "expd_store_state",
    "expd_sweep_kernel_launches",
    "expd_dst",
    "expd_nonlin_hat",
    "expd_set_profiling",
    "expd_sweep_stage_ms",
    "expd_debug_kernel_ms",
    "expd_sweep_pass_ms",
    "expd_solver_step_ms",
    "expd_set_zero_guess",
    "expd_layout_query",
    "expd_a2a_schedule",
    "expd_a2a_schedule_keyed",
    "expd_a2a_execute_host",
    "expd_nccl_unique_id",
    "expd_nccl_comm_init",
    "expd_nccl_comm_destroy",
    "expd_host_comm_create",
    "expd_host_comm_destroy",
    "expd_plan_slab_ipc_handle",
    "expd_plan_set_peer_slabs",
    "expd_plan_enable_peer_stores",
]


class ExpdError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Problem(C.Structure):
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


class _Dist(C.Structure):
    _fields_ = [("rank", C.c_int), ("nranks", C.c_int), ("nccl_comm", C.c_void_p)]


class _Layout(C.Structure):
    _fields_ = [("rank", C.c_int), ("nranks", C.c_int), ("npad", C.c_long), ("mode_off", C.c_long),
                ("mode_len", C.c_long), ("t0", C.c_int), ("nt_local", C.c_int)]


_GroupFn = C.CFUNCTYPE(C.c_int, C.c_void_p)
_SendFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_long, C.c_int)


class _Transport(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("group_start", _GroupFn), ("send", _SendFn), ("recv", _SendFn),
                ("group_end", _GroupFn)]


class _Report(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("sweeps", C.c_int),
        ("converged", C.c_int),
        ("hist_len", C.c_int),
        ("rel_residual", C.c_double),
        ("seconds", C.c_double),
        ("hist", C.POINTER(C.c_double)),
    ]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libexpd.so (raises if it was not built: run paper_2603_04350_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing: build it with `python -m paper_2603_04350_b200.build`")
    lib = C.CDLL(path)
    vp, dp, sz = C.c_void_p, C.POINTER(C.c_double), C.c_size_t
    sig = {
        "expd_plan_create": (C.c_int, [C.POINTER(_Problem), C.POINTER(_Dist), C.c_int, vp, C.POINTER(vp)]),
        "expd_plan_workspace_bytes": (C.c_int, [vp, C.c_int, C.POINTER(sz)]),
        "expd_plan_set_workspace": (C.c_int, [vp, vp, sz]),
        "expd_plan_destroy": (None, [vp]),
        "expd_plan_last_error": (C.c_char_p, [vp]),
        "expd_residual": (C.c_int, [vp, vp, vp, vp, dp]),
        "expd_precond_apply": (C.c_int, [vp, vp, vp]),
        "expd_fixed_point_solve": (C.c_int, [vp, vp, vp, C.c_double, C.c_int, C.POINTER(_Report)]),
        "expd_gmres_solve": (C.c_int, [vp, vp, vp, C.c_double, C.c_int, C.c_int, C.POINTER(_Report)]),
        "expd_bicgstab_solve": (C.c_int, [vp, vp, vp, C.c_double, C.c_int, C.POINTER(_Report)]),
        "expd_load_state": (C.c_int, [vp, vp, vp]),
        "expd_sweep": (C.c_int, [vp]),
        "expd_sweep_norm2": (C.c_int, [vp, dp]),
        "expd_store_state": (C.c_int, [vp, vp]),
        "expd_sweep_kernel_launches": (C.c_int, [vp]),
        "expd_dst": (C.c_int, [vp, vp, vp, C.c_long]),
        "expd_nonlin_hat": (C.c_int, [vp, vp, vp, C.c_long]),
        "expd_set_profiling": (C.c_int, [vp, C.c_int]),
        "expd_sweep_stage_ms": (C.c_int, [vp, dp, dp]),
        "expd_debug_kernel_ms": (C.c_int, [vp, C.c_int, C.c_long, C.c_int, dp]),
        "expd_sweep_pass_ms": (C.c_int, [vp, dp, dp, dp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                         C.POINTER(C.c_int)]),
        "expd_solver_step_ms": (C.c_int, [vp, dp, C.c_int, C.POINTER(C.c_int)]),
        "expd_set_zero_guess": (C.c_int, [vp, C.c_int]),
        "expd_layout_query": (C.c_int, [C.POINTER(_Problem), C.c_int, C.c_int, C.POINTER(_Layout)]),
        "expd_a2a_schedule": (C.c_long, [C.POINTER(_Problem), C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.POINTER(C.c_long), C.POINTER(C.c_long), C.c_long]),
        "expd_a2a_schedule_keyed": (C.c_long, [C.POINTER(_Problem), C.c_int, C.c_int, C.c_int, C.c_int,
                                               C.POINTER(C.c_long), C.POINTER(C.c_long), C.c_long, C.c_int]),
        "expd_a2a_execute_host": (C.c_int, [C.POINTER(_Problem), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.c_int, dp, dp, C.POINTER(_Transport)]),
        "expd_nccl_unique_id": (C.c_int, [C.POINTER(C.c_ubyte)]),
        "expd_nccl_comm_init": (C.c_int, [C.POINTER(C.c_ubyte), C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
        "expd_nccl_comm_destroy": (None, [vp]),
        "expd_host_comm_create": (C.c_int, [C.POINTER(_Transport), C.c_int, C.c_int, C.POINTER(vp)]),
        "expd_host_comm_destroy": (None, [vp]),
        "expd_plan_slab_ipc_handle": (C.c_int, [vp, C.POINTER(C.c_ubyte), C.POINTER(C.c_long), C.POINTER(C.c_long)]),
        "expd_plan_set_peer_slabs": (C.c_int, [vp, C.c_int, C.POINTER(C.c_ubyte), C.c_long, C.c_long]),
        "expd_plan_enable_peer_stores": (C.c_int, [vp, C.c_int]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    _lib = lib
    return lib


@dataclass
class Problem:
    """u_t = (a Delta - c) u + N(u) on (0,1)^dim, Dirichlet, n points/axis, nt steps of dt
    (PAPER.md:53-61, :87-98); N(u) = sum_p q[p] u^p; scheme 0 = exp. Euler / ETD1, 1 = ETD2."""

    dim: int
    n: int
    a: float
    c: float
    dt: float
    nt: int
    alpha: float
    scheme: int = 0
    q: tuple = field(default_factory=tuple)
    a_im: float = 0.0  # imaginary parts of a, c: a complex plan (complex128 vectors, linear only)
    c_im: float = 0.0

    @classmethod
    def from_config(cls, cfg) -> "Problem":
        return cls(cfg.dim, cfg.n, cfg.a, cfg.c, cfg.T / cfg.nt, cfg.nt, cfg.alpha, cfg.scheme, tuple(cfg.q),
                   getattr(cfg, "a_im", 0.0), getattr(cfg, "c_im", 0.0))

    @property
    def is_complex(self) -> bool:
        return self.a_im != 0.0 or self.c_im != 0.0

    @property
    def dtype(self) -> torch.dtype:
        return torch.complex128 if self.is_complex else torch.float64

    @property
    def N(self) -> int:
        return self.n ** self.dim

    @property
    def shape(self) -> tuple:
        return (self.n,) * self.dim

    def _c(self) -> _Problem:
        p = _Problem()
        p.dim, p.n, p.a, p.c, p.dt, p.nt, p.alpha = self.dim, self.n, self.a, self.c, self.dt, self.nt, self.alpha
        p.scheme, p.npoly = self.scheme, len(self.q)
        for i, v in enumerate(self.q):
            p.q[i] = float(v)
        p.a_im, p.c_im = float(self.a_im), float(self.c_im)
        return p


def layout(problem: Problem, rank: int, nranks: int) -> dict:
    """This rank's time slab and mode slab (expd_layout_query; host only, no device)."""
    lib = load_library()
    out = _Layout()
    st = lib.expd_layout_query(C.byref(problem._c()), rank, nranks, C.byref(out))
    if st != EXPD_OK:
        raise ExpdError(st, "expd_layout_query")
    return {k: getattr(out, k) for k, _ in _Layout._fields_}


def a2a_schedule(problem: Problem, rank: int, nranks: int, direction: int, shift: int = 0, keyed: bool = False):
    """The all-to-all messages this rank posts (expd_a2a_schedule): two int64 arrays
    (sends, recvs) of rows {peer, src_off, dst_off, count} (+ slice key when keyed), in
    posting order."""
    import numpy as np

    lib = load_library()
    p = problem._c()
    w = 5 if keyed else 4
    n = lib.expd_a2a_schedule_keyed(C.byref(p), rank, nranks, direction, shift, None, None, 0, w)
    if n < 0:
        raise ExpdError(1, "expd_a2a_schedule")
    s = np.zeros((n, w), dtype=np.int64)
    r = np.zeros((n, w), dtype=np.int64)
    lp = C.POINTER(C.c_long)
    lib.expd_a2a_schedule_keyed(C.byref(p), rank, nranks, direction, shift, s.ctypes.data_as(lp),
                                r.ctypes.data_as(lp), n, w)
    return s, r


def _make_transport(send, recv, group_start=None, group_end=None):
    """An expd_transport over Python callables (numpy views of the message buffers); returns
    the struct and the ctypes callbacks, which must stay referenced while it is in use.  A
    callable that raises reports failure (status 1) to the library."""
    import numpy as np

    def view(ptr, n):
        return np.ctypeslib.as_array(ptr, shape=(int(n),))

    def guard(f):
        def g(*a):
            try:
                return int(f(*a) or 0)
            except Exception:  # an exception must not cross the C frames
                import traceback

                traceback.print_exc()
                return 1
        return g

    cb = [_GroupFn(guard(lambda ctx: group_start() if group_start else 0)),
          _SendFn(guard(lambda ctx, ptr, n, peer: send(view(ptr, n), int(peer)))),
          _SendFn(guard(lambda ctx, ptr, n, peer: recv(view(ptr, n), int(peer)))),
          _GroupFn(guard(lambda ctx: group_end() if group_end else 0))]
    return _Transport(None, *cb), cb


def a2a_execute_host(problem: Problem, rank: int, nranks: int, direction: int, shift: int, src, dst,
                     send, recv, group_start=None, group_end=None, s_lo: int = 0, s_hi: int = 1 << 30):
    """Run this rank's all-to-all (expd_a2a_execute_host) on host float64 numpy arrays with a
    Python transport: send(view, peer) / recv(view, peer) get numpy views of the message
    buffers (valid until group_end() returns); group_start() / group_end() bracket a chunk.
    The library selects, pairs and orders the messages exactly as on the GPU (NCCL)."""
    import numpy as np

    lib = load_library()
    assert src.dtype == np.float64 and dst.dtype == np.float64 and src.flags.c_contiguous and dst.flags.c_contiguous

    tr, cb = _make_transport(send, recv, group_start, group_end)
    dp = C.POINTER(C.c_double)
    st = lib.expd_a2a_execute_host(C.byref(problem._c()), rank, nranks, direction, shift, s_lo, s_hi,
                                   src.ctypes.data_as(dp), dst.ctypes.data_as(dp), C.byref(tr))
    if st != EXPD_OK:
        raise ExpdError(st, "expd_a2a_execute_host")


class Comm:
    """An NCCL communicator for distributed plans.  Rank 0's unique id is
    broadcast over a torch.distributed process group; the library creates the communicator
    (expd_nccl_comm_init) and this object owns it."""

    def __init__(self, rank: int, nranks: int, device: int, group=None):
        import torch.distributed as dist

        self.lib = load_library()
        self.rank, self.nranks, self.device = rank, nranks, device
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            st = self.lib.expd_nccl_unique_id(uid)
            if st != EXPD_OK:
                raise ExpdError(st, "expd_nccl_unique_id")
        if nranks > 1:
            backend = dist.get_backend(group)
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
            if backend == "nccl":
                t = t.to(f"cuda:{device}")
            dist.broadcast(t, src=0, group=group)
            uid = (C.c_ubyte * 128)(*t.cpu().tolist())
        h = C.c_void_p()
        st = self.lib.expd_nccl_comm_init(uid, nranks, rank, device, C.byref(h))
        if st != EXPD_OK:
            raise ExpdError(st, "expd_nccl_comm_init")
        self.ptr = h

    def close(self):
        if getattr(self, "ptr", None):
            self.lib.expd_nccl_comm_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HostComm:
    """A host communicator (expd_host_comm_create) for distributed plans: the plan's
    all-to-alls and allreduces go through host buffers and `transport`, an object with
    send(view, peer), recv(view, peer), group_start(), group_end() (e.g. torch.distributed
    gloo; tests/test_gpu_multirank.py).  Lets several ranks share one GPU; NVLink runs use
    Comm (NCCL)."""

    def __init__(self, rank: int, nranks: int, device: int, transport):
        self.lib = load_library()
        self.rank, self.nranks, self.device = rank, nranks, device
        self._tr, self._cb = _make_transport(transport.send, transport.recv, getattr(transport, "group_start", None),
                                             getattr(transport, "group_end", None))
        h = C.c_void_p()
        st = self.lib.expd_host_comm_create(C.byref(self._tr), rank, nranks, C.byref(h))
        if st != EXPD_OK:
            raise ExpdError(st, "expd_host_comm_create")
        self.ptr = h

    def close(self):
        if getattr(self, "ptr", None):
            self.lib.expd_host_comm_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ptr(t: torch.Tensor | None, dtype: torch.dtype = torch.float64):
    if t is None:
        return None
    if not (t.is_cuda and t.dtype == dtype and t.is_contiguous()):
        raise ValueError(f"expected a contiguous {dtype} CUDA tensor")
    return C.c_void_p(t.data_ptr())


class Plan:
    """An expd_plan plus its torch-allocated workspace on one device."""

    def __init__(self, problem: Problem, device: int | None = None, krylov_vectors: int = 0, stream=None,
                 comm: Comm | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("expd requires a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.problem = problem
        self.device = torch.cuda.current_device() if device is None else device
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._p = problem._c()
        # comm: distributed schedule (time slabs in the API, mode slabs for K1); with
        # comm.nranks == 1 it runs on one GPU with local copies for the all-to-alls
        self.comm = comm
        dist = _Dist(comm.rank, comm.nranks, comm.ptr) if comm is not None else _Dist(0, 1, None)
        self.layout = layout(problem, dist.rank, dist.nranks)
        handle = C.c_void_p()
        st = self.lib.expd_plan_create(C.byref(self._p), C.byref(dist), self.device,
                                       C.c_void_p(self.stream.cuda_stream), C.byref(handle))
        if st != EXPD_OK:
            raise ExpdError(st, "expd_plan_create")
        self.handle = handle
        nbytes = C.c_size_t()
        self._check(self.lib.expd_plan_workspace_bytes(self.handle, krylov_vectors, C.byref(nbytes)))
        self.workspace = torch.empty(nbytes.value + 256, dtype=torch.uint8, device=f"cuda:{self.device}")
        base = self.workspace.data_ptr()
        aligned = (base + 255) // 256 * 256
        self._check(self.lib.expd_plan_set_workspace(self.handle, C.c_void_p(aligned), nbytes.value))

    def _check(self, st: int):
        if st != EXPD_OK:
            msg = self.lib.expd_plan_last_error(self.handle).decode() if getattr(self, "handle", None) else ""
            raise ExpdError(st, msg)

    def close(self):
        if getattr(self, "handle", None):
            self.lib.expd_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _vec(self):
        """A physical space-time vector of this rank: its time slab (all nt slices on one GPU)."""
        return torch.empty((self.layout["nt_local"],) + self.problem.shape, dtype=self.problem.dtype,
                           device=f"cuda:{self.device}")

    def _a(self, t, slices: int | None = None):
        """A state argument (u0, U, R, S): float64, or complex128 for a complex plan, on the
        plan's device, holding `slices` spatial slices (default: this rank's time slab; 1 for
        u0).  The C-ABI reads / writes exactly that many elements through the raw pointer, so
        a wrong shape or device is rejected here instead of faulting on the device."""
        if t is None:
            return None
        want = (self.layout["nt_local"] if slices is None else slices) * self.problem.N
        return self._chk(t, self.problem.dtype, want)

    def _chk(self, t, dtype, numel: int, host_ok: bool = False):
        if not isinstance(t, torch.Tensor):
            raise ValueError("expected a torch tensor")
        if t.numel() != numel:
            raise ValueError(f"tensor holds {t.numel()} elements, expected {numel}")
        if host_ok and t.device.type == "cpu":  # solver I/O with host buffers (single-GPU plans)
            if not (t.dtype == dtype and t.is_contiguous()):
                raise ValueError(f"expected a contiguous {dtype} tensor")
            return C.c_void_p(t.data_ptr())
        if t.device.type != "cuda" or t.device.index != self.device:
            raise ValueError(f"tensor on {t.device}, plan on cuda:{self.device}")
        return _ptr(t, dtype)

    def _io(self, t, slices: int | None = None):
        """A solver argument (u0, U): on the plan's device, or a host tensor (pinned for
        overlapped copies) that the library copies in / streams out itself."""
        want = (self.layout["nt_local"] if slices is None else slices) * self.problem.N
        return self._chk(t, self.problem.dtype, want, host_ok=self.comm is None)

    def enable_peer_stores(self, group=None):
        """Stage 3 of this distributed plan loads its rows straight from the owners' U-hat slabs
        and stores them straight into the owners' N-hat slabs (expd_plan_*slab* / *peer*: CUDA
        IPC handles exchanged over torch.distributed, collective over the plan's ranks)."""
        import torch.distributed as dist

        h = (C.c_ubyte * 64)()
        offn, offu = C.c_long(), C.c_long()
        self._check(self.lib.expd_plan_slab_ipc_handle(self.handle, h, C.byref(offn), C.byref(offu)))
        allh = [None] * self.comm.nranks
        dist.all_gather_object(allh, (bytes(h), offn.value, offu.value), group=group)
        for q, (hb, on, ou) in enumerate(allh):
            self._check(self.lib.expd_plan_set_peer_slabs(self.handle, q, (C.c_ubyte * 64)(*hb), on, ou))
        self._check(self.lib.expd_plan_enable_peer_stores(self.handle, 1))

    def set_zero_guess(self, on: bool = True):
        """Solvers start from U = 0 and ignore U's contents on entry."""
        self._check(self.lib.expd_set_zero_guess(self.handle, int(bool(on))))

    # ---- primitives ------------------------------------------------------------------
    def residual(self, u0: torch.Tensor, U: torch.Tensor, R: torch.Tensor | None = None, norm: bool = False):
        R = self._vec() if R is None else R
        rn = C.c_double()
        self._check(self.lib.expd_residual(self.handle, self._a(u0, 1), self._a(U), self._a(R),
                                           C.pointer(rn) if norm else None))
        return (R, rn.value) if norm else R

    def precond_apply(self, R: torch.Tensor, S: torch.Tensor | None = None):
        S = self._vec() if S is None else S
        self._check(self.lib.expd_precond_apply(self.handle, self._a(R), self._a(S)))
        return S

    # ---- solvers ---------------------------------------------------------------------
    def _report(self, maxit):
        hist = (C.c_double * (maxit + 2))()
        r = _Report()
        r.hist = C.cast(hist, C.POINTER(C.c_double))
        return r, hist

    @staticmethod
    def _rdict(r, hist, status):
        return {
            "status": STATUS.get(status, status),
            "iterations": r.iterations,
            "sweeps": r.sweeps,
            "converged": bool(r.converged),
            "rel_residual": r.rel_residual,
            "seconds": r.seconds,
            "hist": [hist[i] for i in range(r.hist_len)],
        }

    def fixed_point_solve(self, u0, U=None, tol=1e-12, maxit=100):
        U = self._vec().zero_() if U is None else U
        r, hist = self._report(maxit)
        st = self.lib.expd_fixed_point_solve(self.handle, self._io(u0, 1), self._io(U), tol, maxit, C.byref(r))
        if st not in (EXPD_OK, 7):
            self._check(st)
        return U, self._rdict(r, hist, st)

    def gmres_solve(self, u0, U=None, tol=1e-12, restart=20, maxit=100):
        U = self._vec().zero_() if U is None else U
        r, hist = self._report(maxit)
        st = self.lib.expd_gmres_solve(self.handle, self._io(u0, 1), self._io(U), tol, restart, maxit, C.byref(r))
        if st not in (EXPD_OK, 7):
            self._check(st)
        return U, self._rdict(r, hist, st)

    def bicgstab_solve(self, u0, U=None, tol=1e-12, maxit=100):
        U = self._vec().zero_() if U is None else U
        r, hist = self._report(maxit)
        st = self.lib.expd_bicgstab_solve(self.handle, self._io(u0, 1), self._io(U), tol, maxit, C.byref(r))
        if st not in (EXPD_OK, 7):
            self._check(st)
        return U, self._rdict(r, hist, st)

    # ---- spectral-state sweep (benchmark / fine-grained driving) ----------------------
    def load_state(self, u0, U=None):
        self._check(self.lib.expd_load_state(self.handle, self._a(u0, 1), self._a(U)))

    def sweep(self):
        self._check(self.lib.expd_sweep(self.handle))

    def sweep_norm2(self) -> float:
        v = C.c_double()
        self._check(self.lib.expd_sweep_norm2(self.handle, C.byref(v)))
        return v.value

    def store_state(self, U):
        self._check(self.lib.expd_store_state(self.handle, self._a(U)))

    def dst(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """V x for a stack of physical slices [..., n, ..., n]."""
        out = torch.empty_like(x) if out is None else out
        ns = x.numel() // self.problem.N
        if ns * self.problem.N != x.numel():
            raise ValueError("x must hold whole slices of n^dim points")
        if ns == 0:
            return out
        self._check(self.lib.expd_dst(self.handle, self._chk(x, torch.float64, x.numel()),
                                      self._chk(out, torch.float64, x.numel()), ns))
        return out

    def nonlin_hat(self, uhat: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """V N(V uhat) for a stack of DST-coefficient slices [..., n, ..., n] (stage 3)."""
        out = torch.empty_like(uhat) if out is None else out
        ns = uhat.numel() // self.problem.N
        if ns * self.problem.N != uhat.numel():
            raise ValueError("uhat must hold whole slices of n^dim points")
        if ns == 0:
            return out
        self._check(self.lib.expd_nonlin_hat(self.handle, self._chk(uhat, torch.float64, uhat.numel()),
                                             self._chk(out, torch.float64, uhat.numel()), ns))
        return out

    def set_profiling(self, enable: bool | int = True):
        """0 off, 1 (True) stage events, 2 stage events + an event between stage-3 passes."""
        self._check(self.lib.expd_set_profiling(self.handle, int(enable)))

    def sweep_stage_ms(self):
        """(stage-3 ms, K1 ms) of the last sweep (device time, CUDA events)."""
        a, b = C.c_double(), C.c_double()
        self._check(self.lib.expd_sweep_stage_ms(self.handle, C.byref(a), C.byref(b)))
        return a.value, b.value

    def sweep_pass_ms(self) -> dict:
        """Stage-3 pass times of the last sweep, from events inside the sweep (profiling on)."""
        t = [C.c_double() for _ in range(3)]
        n = [C.c_int() for _ in range(3)]
        self._check(self.lib.expd_sweep_pass_ms(self.handle, *(C.byref(x) for x in t), *(C.byref(x) for x in n)))
        return {"x_ms": t[0].value, "strided_ms": t[1].value, "fused_ms": t[2].value,
                "x_launches": n[0].value, "strided_launches": n[1].value, "fused_launches": n[2].value}

    def solver_step_ms(self) -> list:
        """Device ms of every Arnoldi step of the last GMRES solve (profiling on)."""
        n = C.c_int()
        self._check(self.lib.expd_solver_step_ms(self.handle, None, 0, C.byref(n)))
        buf = (C.c_double * max(n.value, 1))()
        self._check(self.lib.expd_solver_step_ms(self.handle, buf, n.value, C.byref(n)))
        return [buf[i] for i in range(n.value)]

    def debug_kernel_ms(self, which: int, nslices: int = 1, reps: int = 10) -> float:
        v = C.c_double()
        self._check(self.lib.expd_debug_kernel_ms(self.handle, which, nslices, reps, C.byref(v)))
        return v.value

    def sweep_kernel_launches(self) -> int:
        return int(self.lib.expd_sweep_kernel_launches(self.handle))
