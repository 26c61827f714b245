"""Thin ctypes binding of libhmg.so (include/hmg.h).

Argument marshalling only: every step of the method runs in the library's CUDA
kernels.  Vectors are torch CUDA tensors (complex64 / complex128, contiguous,
x-fastest node order, i.e. numpy/torch shape ``nodes[::-1]`` or flat); the
binding passes their device pointers and the current torch stream.  There is
NO CPU fallback: importing this module on a machine without the built library
raises, and every call raises ``HmgError`` on a non-OK status.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhmg.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2511_16808_b200.build` "
                      "(the CUDA path has no fallback)")
_lib = ctypes.CDLL(LIB_PATH)

# enums (include/hmg.h)
OK, EINVAL, ESINGULAR_PATCH, ESINGULAR_COARSE, EBREAKDOWN, ENOTCONVERGED, ENOMEM, ECUDA, ENCCL = range(9)
C64, C128 = 0, 1
COMPACT4, FD2 = 0, 1
LEVDEP, LINEAR, CUBIC, MIXED = 0, 1, 2, 3
GALERKIN, REDISCRETIZE = 0, 1
VANKA_RB, VANKA_ELEMENT, JACOBI, VANKA_PLUS = 0, 1, 2, 3

STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "ESINGULAR_PATCH", 3: "ESINGULAR_COARSE", 4: "EBREAKDOWN",
                5: "ENOTCONVERGED", 6: "ENOMEM", 7: "ECUDA", 8: "ENCCL"}
_NAMES = {
    "compact4": COMPACT4, "fd2": FD2,
    "levdep": LEVDEP, "linear": LINEAR, "cubic": CUBIC, "mixed": MIXED,
    "galerkin": GALERKIN, "rediscretize": REDISCRETIZE,
    "rb": VANKA_RB, "element": VANKA_ELEMENT, "jacobi": JACOBI, "plus": VANKA_PLUS,
}


class _Options(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("cells", ctypes.c_int64 * 3), ("h", ctypes.c_double),
                ("levels", ctypes.c_int), ("nu1", ctypes.c_int), ("nu2", ctypes.c_int),
                ("cycle", ctypes.c_int), ("fine_stencil", ctypes.c_int), ("intergrid", ctypes.c_int),
                ("coarse_op", ctypes.c_int), ("smoother", ctypes.c_int),
                ("damping", ctypes.POINTER(ctypes.c_double)), ("n_damping", ctypes.c_int),
                ("dtype", ctypes.c_int)]


class _Report(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("converged", ctypes.c_int), ("restarts", ctypes.c_int),
                ("history_len", ctypes.c_int), ("history_cap", ctypes.c_int),
                ("history", ctypes.POINTER(ctypes.c_double)), ("relres_true", ctypes.c_double),
                ("relres_est", ctypes.c_double), ("c_f", ctypes.c_double), ("seconds", ctypes.c_double)]


_vp, _i, _d, _i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int64
_sigs = {
    "hmg_build_hierarchy": ([ctypes.POINTER(_Options), _vp, _d, _vp, _d, _vp, ctypes.POINTER(_vp)], _i),
    "hmg_apply_helmholtz": ([_vp, _i, _i, _vp, _vp, _vp], _i),
    "hmg_residual": ([_vp, _i, _i, _vp, _vp, _vp, _vp], _i),
    "hmg_smooth": ([_vp, _i, _vp, _vp, _vp], _i),
    "hmg_restrict": ([_vp, _i, _vp, _vp, _vp], _i),
    "hmg_prolong_add": ([_vp, _i, _vp, _vp, _vp], _i),
    "hmg_coarse_solve": ([_vp, _vp, _vp, _vp], _i),
    "hmg_vcycle": ([_vp, _vp, _vp, _i, _vp], _i),
    "hmg_fgmres_solve": ([_vp, _vp, _vp, _i, _d, _i, _vp, ctypes.POINTER(_Report)], _i),
    "hmg_fgmres_solve_host": ([_vp, _vp, _vp, _i, _d, _i, _vp, ctypes.POINTER(_Report)], _i),
    "hmg_fgmres_solve_batch": ([_vp, _i, _vp, _vp, _i, _d, _i, _vp, ctypes.POINTER(_Report)], _i),
    "hmg_num_levels": ([_vp], _i),
    "hmg_level_nodes": ([_vp, _i, ctypes.POINTER(_i64)], _i64),
    "hmg_stencil_radius": ([_vp, _i], _i),
    "hmg_copy_stencil": ([_vp, _i, ctypes.POINTER(_d), _i64], _i),
    "hmg_uniform_box": ([_vp, _i, ctypes.POINTER(_i64), ctypes.POINTER(_i64)], _i64),
    "hmg_dict_classes": ([_vp, _i, ctypes.POINTER(_i), ctypes.POINTER(_i)], _i),
    "hmg_launch_count": ([], _i64),
    "hmg_profile_begin": ([], None),
    "hmg_profile_report": ([], ctypes.c_char_p),
    "hmg_hierarchy_destroy": ([_vp], None),
    "hmg_comm_local_group": ([_i, ctypes.POINTER(_vp)], _i),
    "hmg_comm_local_rank": ([_vp, _i, ctypes.POINTER(_vp)], _i),
    "hmg_comm_nccl_unique_id": ([_vp], _i),
    "hmg_comm_nccl": ([_vp, _i, _i, ctypes.POINTER(_vp)], _i),
    "hmg_comm_destroy": ([_vp], None),
    "hmg_build_hierarchy_dist": ([ctypes.POINTER(_Options), _vp, _d, _vp, _d, _vp, _vp, ctypes.POINTER(_vp)], _i),
    "hmg_level_rows": ([_vp, _i, ctypes.POINTER(_i64), ctypes.POINTER(_i64)], _i),
    "hmg_setup_plan": ([ctypes.POINTER(_Options), _i, _i, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                        ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_d)], _i),
    "hmg_slab_partition": ([_i64, _i, _i, _i, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i)], _i),
    "hmg_last_error": ([], ctypes.c_char_p),
    "hmg_version": ([], ctypes.c_char_p),
}
for _n, (_a, _r) in _sigs.items():
    _f = getattr(_lib, _n)
    _f.argtypes = _a
    _f.restype = _r

EXPORTED = tuple(_sigs)


class HmgError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _check(st):
    if st != OK:
        raise HmgError(st, _lib.hmg_last_error().decode())


def last_error():
    return _lib.hmg_last_error().decode()


def launch_count():
    return int(_lib.hmg_launch_count())


def profile_begin():
    """Start per-kernel CUDA-event timing inside the library (hmg_profile_begin)."""
    _lib.hmg_profile_begin()


def profile_report():
    """Stop timing; {kernel@Llevel: {launches, ms, bytes}} (hmg_profile_report)."""
    import json
    return json.loads(_lib.hmg_profile_report().decode())


def version():
    return _lib.hmg_version().decode()


def _stream(stream):
    if stream is not None:
        return ctypes.c_void_p(int(getattr(stream, "cuda_stream", stream)))
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t, dtype, n):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("expected a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {t.dtype}")
    if not t.is_contiguous() or t.numel() != n:
        raise ValueError(f"expected a contiguous tensor of {n} elements, got shape {tuple(t.shape)}")
    return ctypes.c_void_p(t.data_ptr())


class Comm:
    """A rank's communicator (hmg_comm).  Build with ``LocalGroup(k).rank(r)``
    (k virtual ranks on one GPU, one host thread each) or ``Comm.nccl(uid, rank, n)``."""

    def __init__(self, handle, rank, size, keep=None):
        self._h, self.rank, self.size, self._keep = handle, rank, size, keep

    @staticmethod
    def nccl_unique_id():
        buf = (ctypes.c_char * 128)()
        _check(_lib.hmg_comm_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
        return bytes(buf)

    @classmethod
    def nccl(cls, uid, rank, size):
        buf = (ctypes.c_char * 128).from_buffer_copy(uid)
        h = ctypes.c_void_p()
        _check(_lib.hmg_comm_nccl(ctypes.cast(buf, ctypes.c_void_p), rank, size, ctypes.byref(h)))
        return cls(h, rank, size)

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.hmg_comm_destroy(self._h)
            self._h = None


class LocalGroup:
    """k virtual ranks on the current GPU (hmg_comm_local_group)."""

    def __init__(self, size):
        h = ctypes.c_void_p()
        _check(_lib.hmg_comm_local_group(size, ctypes.byref(h)))
        self._h, self.size = h, size

    def rank(self, r):
        h = ctypes.c_void_p()
        _check(_lib.hmg_comm_local_rank(self._h, r, ctypes.byref(h)))
        return Comm(h, r, self.size, keep=self)

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.hmg_comm_destroy(self._h)
            self._h = None


def setup_plan(opts, nranks, rank):
    """Host-only memory plan of the partitioned build (hmg_setup_plan): dict with per-level
    setup windows and kept rows, and the modelled peak / resident / FGMRES(20) bytes."""
    o = opts.to_c()
    L = opts.levels
    arr = [(ctypes.c_int64 * L)() for _ in range(4)]
    b = (ctypes.c_double * 3)()
    nd = _lib.hmg_setup_plan(ctypes.byref(o), nranks, rank, *arr, b)
    if nd < 0:
        raise HmgError(EINVAL, "bad arguments")
    wlo, whi, klo, khi = ([int(v) for v in a] for a in arr)
    return {"partitioned_levels": nd, "window": list(zip(wlo, whi)), "kept": list(zip(klo, khi)),
            "setup_peak_bytes": b[0], "resident_bytes": b[1], "fgmres20_bytes": b[2]}


def slab_partition(nodes0, levels, nranks, ghost=4):
    """Host-only partition rule (hmg_slab_partition): (lo, hi) arrays [levels, nranks], dist [levels]."""
    lo = (ctypes.c_int64 * (levels * nranks))()
    hi = (ctypes.c_int64 * (levels * nranks))()
    dist = (ctypes.c_int * levels)()
    n = _lib.hmg_slab_partition(nodes0, levels, nranks, ghost, lo, hi, dist)
    if n < 0:
        raise HmgError(EINVAL, "bad partition arguments")
    return (np.array(lo[:]).reshape(levels, nranks), np.array(hi[:]).reshape(levels, nranks),
            np.array(dist[:]))


@dataclass
class Report:
    iterations: int
    converged: bool
    restarts: int
    history: list
    relres_true: float
    relres_est: float
    c_f: float
    seconds: float
    status: int = OK


@dataclass
class Options:
    dim: int
    cells: tuple
    h: float
    levels: int = 4
    nu1: int = 1
    nu2: int = 1
    cycle: str = "V"
    fine_stencil: str = "compact4"
    intergrid: str = "levdep"
    coarse_op: str = "galerkin"
    smoother: str = "rb"
    damping: list = field(default_factory=lambda: [0.83, 0.5, 0.4, 0.65])
    dtype: str = "c128"

    def to_c(self):
        """The hmg_options struct (marshalling only); keeps the damping array alive on it."""
        o = _Options()
        o.dim = self.dim
        cells = list(self.cells) + [0] * (3 - len(self.cells))
        for a in range(3):
            o.cells[a] = int(cells[a])
        o.h = float(self.h)
        o.levels = int(self.levels)
        o.nu1, o.nu2 = int(self.nu1), int(self.nu2)
        o.cycle = {"V": 0, "W": 1}[self.cycle]
        o.fine_stencil = _NAMES[self.fine_stencil]
        o.intergrid = _NAMES[self.intergrid]
        o.coarse_op = _NAMES[self.coarse_op]
        o.smoother = _NAMES[self.smoother]
        o._damp = (ctypes.c_double * len(self.damping))(*[float(x) for x in self.damping])
        o.damping = ctypes.cast(o._damp, ctypes.POINTER(ctypes.c_double))
        o.n_damping = len(self.damping)
        o.dtype = {"c64": C64, "c128": C128}[self.dtype]
        return o


class Hierarchy:
    """Owns an hmg_hierarchy handle (hmg_build_hierarchy ... hmg_hierarchy_destroy)."""

    def __init__(self, opts: Options, kappa, omega, gamma, alpha, stream=None, comm: "Comm" = None):
        import torch
        o = opts.to_c()
        self._o = o
        self.opts = opts
        self.dtype = torch.complex64 if opts.dtype == "c64" else torch.complex128
        k = np.ascontiguousarray(np.asarray(kappa, dtype=np.float64).ravel())
        g = np.ascontiguousarray(np.asarray(gamma, dtype=np.float64).ravel())
        nodes = [c + 1 for c in opts.cells]
        if k.size != int(np.prod(nodes)) or g.size != k.size:
            raise ValueError("kappa/gamma size does not match the grid")
        h = ctypes.c_void_p()
        self._h = None
        self.comm = comm
        if comm is None:
            _check(_lib.hmg_build_hierarchy(ctypes.byref(o), k.ctypes.data_as(ctypes.c_void_p), float(omega),
                                            g.ctypes.data_as(ctypes.c_void_p), float(alpha), _stream(stream),
                                            ctypes.byref(h)))
        else:
            _check(_lib.hmg_build_hierarchy_dist(ctypes.byref(o), k.ctypes.data_as(ctypes.c_void_p), float(omega),
                                                 g.ctypes.data_as(ctypes.c_void_p), float(alpha), comm._h,
                                                 _stream(stream), ctypes.byref(h)))
        self._h = h
        self.levels = int(_lib.hmg_num_levels(h))

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.hmg_hierarchy_destroy(self._h)
            self._h = None

    # ---------------------------------------------------------------- info
    def level_nodes(self, level):
        n = (ctypes.c_int64 * 3)()
        N = _lib.hmg_level_nodes(self._h, level, n)
        if N < 0:
            raise HmgError(EINVAL, "level out of range")
        return int(N), tuple(int(n[a]) for a in range(self.opts.dim))

    def level_rows(self, level):
        """Global slab-axis rows [lo, hi) this rank holds on ``level``."""
        lo, hi = ctypes.c_int64(), ctypes.c_int64()
        if _lib.hmg_level_rows(self._h, level, ctypes.byref(lo), ctypes.byref(hi)) != 0:
            raise HmgError(EINVAL, "level out of range")
        return lo.value, hi.value

    def uniform_box(self, level):
        """(nodes, lo, hi) of the level's uniform-coefficient box."""
        lo, hi = (ctypes.c_int64 * 3)(), (ctypes.c_int64 * 3)()
        n = _lib.hmg_uniform_box(self._h, level, lo, hi)
        if n < 0:
            raise HmgError(EINVAL, "level out of range")
        return int(n), tuple(lo[a] for a in range(self.opts.dim)), tuple(hi[a] for a in range(self.opts.dim))

    def dict_classes(self, level):
        """(stencil classes, Vanka-operator classes) of the level's coefficient
        dictionaries; 0 where the planes are read."""
        cn, bn = ctypes.c_int(), ctypes.c_int()
        if _lib.hmg_dict_classes(self._h, level, ctypes.byref(cn), ctypes.byref(bn)) != 0:
            raise HmgError(EINVAL, "level out of range")
        return cn.value, bn.value

    def stencil_radius(self, level):
        return int(_lib.hmg_stencil_radius(self._h, level))

    def copy_stencil(self, level):
        """Level operator as complex128 array [K, N] (offsets x-fastest in -r..r)."""
        N, _ = self.level_nodes(level)
        r = self.stencil_radius(level)
        K = (2 * r + 1) ** self.opts.dim
        out = np.zeros(2 * K * N, np.float64)
        k = _lib.hmg_copy_stencil(self._h, level, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), out.size)
        if k < 0:
            raise HmgError(EINVAL, last_error())
        return out.view(np.complex128).reshape(K, N)

    def _n(self, level):
        return self.level_nodes(level)[0]

    # ---------------------------------------------------------------- ops
    def apply_helmholtz(self, x, y, level=0, shifted=False, stream=None):
        n = self._n(level)
        _check(_lib.hmg_apply_helmholtz(self._h, level, int(shifted), _ptr(x, self.dtype, n),
                                        _ptr(y, self.dtype, n), _stream(stream)))

    def residual(self, f, x, r, level=0, shifted=False, stream=None):
        n = self._n(level)
        _check(_lib.hmg_residual(self._h, level, int(shifted), _ptr(f, self.dtype, n), _ptr(x, self.dtype, n),
                                 _ptr(r, self.dtype, n), _stream(stream)))

    def smooth(self, f, u, level=0, stream=None):
        n = self._n(level)
        _check(_lib.hmg_smooth(self._h, level, _ptr(f, self.dtype, n), _ptr(u, self.dtype, n), _stream(stream)))

    def restrict(self, r, fc, level=0, stream=None):
        _check(_lib.hmg_restrict(self._h, level, _ptr(r, self.dtype, self._n(level)),
                                 _ptr(fc, self.dtype, self._n(level + 1)), _stream(stream)))

    def prolong_add(self, ec, u, level=0, stream=None):
        _check(_lib.hmg_prolong_add(self._h, level, _ptr(ec, self.dtype, self._n(level + 1)),
                                    _ptr(u, self.dtype, self._n(level)), _stream(stream)))

    def coarse_solve(self, r, e, stream=None):
        n = self._n(self.levels - 1)
        _check(_lib.hmg_coarse_solve(self._h, _ptr(r, self.dtype, n), _ptr(e, self.dtype, n), _stream(stream)))

    def vcycle(self, f, x, x_is_zero=True, stream=None):
        n = self._n(0)
        _check(_lib.hmg_vcycle(self._h, _ptr(f, self.dtype, n), _ptr(x, self.dtype, n), int(x_is_zero),
                               _stream(stream)))

    def fgmres_solve(self, q, x, restart=10, tol=1e-6, maxiter=500, stream=None, history_cap=100000):
        """Solve H x = q on the device (q, x CUDA tensors).  Returns a Report;
        ENOTCONVERGED is reported in Report.status, other errors raise."""
        n = self._n(0)
        return self._solve(_lib.hmg_fgmres_solve, _ptr(q, self.dtype, n), _ptr(x, self.dtype, n),
                           restart, tol, maxiter, stream, history_cap)

    def fgmres_solve_host(self, q, x, restart=10, tol=1e-6, maxiter=500, stream=None, history_cap=100000):
        """Same with q, x in host memory (torch CPU tensors, ideally pinned)."""
        n = self._n(0)
        for t in (q, x):
            if t.is_cuda or t.dtype != self.dtype or not t.is_contiguous() or t.numel() != n:
                raise ValueError("expected contiguous host tensors of the hierarchy's dtype and size")
        return self._solve(_lib.hmg_fgmres_solve_host, ctypes.c_void_p(q.data_ptr()),
                           ctypes.c_void_p(x.data_ptr()), restart, tol, maxiter, stream, history_cap)

    def fgmres_solve_batch(self, q, x, restart=10, tol=1e-6, maxiter=500, stream=None, history_cap=20000):
        """nrhs independent solves H x_k = q_k on this hierarchy, advanced in lockstep
        with one batched preconditioner per step (hmg_fgmres_solve_batch).  q, x: CUDA
        tensors of shape (nrhs, N) (or nrhs * N contiguous).  Returns a list of Reports."""
        n = self._n(0)
        if q.numel() % n or q.numel() != x.numel():
            raise ValueError("q and x must hold nrhs * N values")
        nr = q.numel() // n
        _ptr(q.view(-1), self.dtype, nr * n)   # contiguous CUDA tensors of the hierarchy's dtype
        _ptr(x.view(-1), self.dtype, nr * n)
        hists = [(ctypes.c_double * history_cap)() for _ in range(nr)]
        reps = (_Report * nr)()
        for k in range(nr):
            reps[k].history = ctypes.cast(hists[k], ctypes.POINTER(ctypes.c_double))
            reps[k].history_cap = history_cap
        st = _lib.hmg_fgmres_solve_batch(self._h, nr, ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(x.data_ptr()),
                                         int(restart), float(tol), int(maxiter), _stream(stream), reps)
        if st not in (OK, ENOTCONVERGED):
            _check(st)
        return [Report(iterations=r.iterations, converged=bool(r.converged), restarts=r.restarts,
                       history=list(h[:r.history_len]), relres_true=r.relres_true, relres_est=r.relres_est,
                       c_f=r.c_f, seconds=r.seconds, status=OK if r.converged else ENOTCONVERGED)
                for r, h in zip(reps, hists)]

    def _solve(self, fn, qp, xp, restart, tol, maxiter, stream, history_cap):
        hist = (ctypes.c_double * history_cap)()
        rep = _Report()
        rep.history = ctypes.cast(hist, ctypes.POINTER(ctypes.c_double))
        rep.history_cap = history_cap
        st = fn(self._h, qp, xp, int(restart), float(tol), int(maxiter), _stream(stream), ctypes.byref(rep))
        if st not in (OK, ENOTCONVERGED):
            _check(st)
        return Report(iterations=rep.iterations, converged=bool(rep.converged), restarts=rep.restarts,
                      history=list(hist[:rep.history_len]), relres_true=rep.relres_true,
                      relres_est=rep.relres_est, c_f=rep.c_f, seconds=rep.seconds, status=st)
