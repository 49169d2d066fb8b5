"""paper_2408_11929_b200 -- B200 (sm_100a) hot path of multipreconditioned
GMRES with directional double-sweep preconditioners for the 2D impedance
Helmholtz problem (Bootland & Rees, arXiv 2408.11929).

This module is a thin ctypes binding over the C ABI declared in
``include/helmsweep.h`` (argument marshalling only).  Every step of the path
runs in the CUDA kernels of ``libhelmsweep.so``; there is no CPU fallback:
importing without the built library, or calling without a CUDA device,
raises.  Vectors are complex128 torch tensors on the GPU (the device path) or
numpy arrays on the host (the end-to-end path: the library stages them).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HELM_LIB") or os.path.join(_HERE, "libhelmsweep.so")

HELM_OK = 0
STATUS = {0: "HELM_OK", 1: "HELM_EINVAL", 2: "HELM_EDIM", 3: "HELM_ESINGULAR", 4: "HELM_ECUDA",
          5: "HELM_ENOMEM", 6: "HELM_ENOCONV", 7: "HELM_EEXHAUSTED", 8: "HELM_ENONFINITE"}

DIRECTIONS = {"LRL": (0, 0, 1), "RLR": (0, 1, 1), "BTB": (1, 0, 1), "TBT": (1, 1, 1),
              "LR": (0, 0, 0), "RL": (0, 1, 0), "BT": (1, 0, 0), "TB": (1, 1, 0)}

EXPORTS = ["helm_assemble", "helm_assemble_fd5", "helm_problem_info", "helm_get_diagonals", "helm_load_vector", "helm_spmv",
           "sweep_setup", "sweep_info", "sweep_apply", "mpgmres_solve", "helm_problem_destroy",
           "sweep_destroy", "helm_strerror", "helm_last_error", "helm_kernel_launches", "helm_sweep_kernel_name",
           "helm_set_knob", "mpgmres_solve_dist", "sweep_set_precision"]


class HelmError(RuntimeError):
    def __init__(self, code, where):
        self.code = code
        super().__init__(f"{where}: {STATUS.get(code, code)}: {last_error()}")


class _GridDesc(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("h", ctypes.c_double),
                ("omega", ctypes.c_double), ("c_nodes", ctypes.c_void_p)]


class MPGMRESStats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("converged", ctypes.c_int), ("flags", ctypes.c_int),
                ("deflations", ctypes.c_int), ("proj_rel_res", ctypes.c_double),
                ("true_rel_res", ctypes.c_double), ("solve_s", ctypes.c_double),
                ("sweep_ms", ctypes.c_double), ("spmv_ms", ctypes.c_double), ("orth_ms", ctypes.c_double),
                ("matvecs", ctypes.c_long), ("prec_applies", ctypes.c_long),
                ("inner_products", ctypes.c_long), ("history", ctypes.POINTER(ctypes.c_double)),
                ("history_cap", ctypes.c_int)]


_lib = None

# helm_allgather_fn (helmsweep.h): int (*)(void* ctx, const void* send, void* recv, long bytes, void* stream)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long,
                                ctypes.c_void_p)


def load():
    """Load libhelmsweep.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2408_11929_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i, d, l = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_long
    L.helm_assemble.argtypes = [ctypes.POINTER(_GridDesc), vp, ctypes.POINTER(vp)]
    L.helm_assemble_fd5.argtypes = [ctypes.POINTER(_GridDesc), vp, ctypes.POINTER(vp)]
    L.helm_problem_info.argtypes = [vp, ctypes.POINTER(l), ctypes.POINTER(i), ctypes.POINTER(i)]
    L.helm_get_diagonals.argtypes = [vp, vp, vp]
    L.helm_load_vector.argtypes = [vp, vp, vp, vp]
    L.helm_spmv.argtypes = [vp, vp, vp, i, vp]
    L.sweep_setup.argtypes = [vp, i, i, i, i, i, i, i, vp, ctypes.POINTER(vp)]
    L.sweep_info.argtypes = [vp, ctypes.POINTER(l)]
    L.sweep_set_precision.argtypes = [vp, i]
    L.sweep_set_precision.restype = i
    L.sweep_apply.argtypes = [ctypes.POINTER(vp), i, vp, l, vp, l, vp]
    L.mpgmres_solve.argtypes = [vp, ctypes.POINTER(vp), i, vp, vp, d, i, ctypes.POINTER(MPGMRESStats), vp]
    L.helm_problem_destroy.argtypes = [vp]
    L.helm_problem_destroy.restype = None
    L.sweep_destroy.argtypes = [vp]
    L.sweep_destroy.restype = None
    L.helm_strerror.argtypes = [i]
    L.helm_strerror.restype = ctypes.c_char_p
    L.helm_last_error.argtypes = []
    L.helm_last_error.restype = ctypes.c_char_p
    L.helm_kernel_launches.argtypes = []
    L.helm_kernel_launches.restype = l
    L.helm_sweep_kernel_name.argtypes = []
    L.helm_sweep_kernel_name.restype = ctypes.c_char_p
    L.helm_set_knob.argtypes = [ctypes.c_char_p, i]
    L.helm_set_knob.restype = i
    L.mpgmres_solve_dist.argtypes = [vp, ctypes.POINTER(vp), i, i, i, ALLGATHER_FN, vp, vp, vp, d, i,
                                     ctypes.POINTER(MPGMRESStats), vp]
    L.mpgmres_solve_dist.restype = i
    for name in ["helm_assemble", "helm_assemble_fd5", "helm_problem_info", "helm_get_diagonals", "helm_load_vector", "helm_spmv",
                 "sweep_setup", "sweep_info", "sweep_apply", "mpgmres_solve"]:
        getattr(L, name).restype = i
    _lib = L
    return L


def last_error() -> str:
    return load().helm_last_error().decode()


def kernel_launches() -> int:
    return int(load().helm_kernel_launches())


def sweep_kernel_name() -> str:
    """Sweep kernel launched by the last apply (diagnostics)."""
    return load().helm_sweep_kernel_name().decode()


def set_knob(name: str, value: int) -> None:
    """helm_set_knob: diagnostics / testing controls (0 = the product choice)."""
    _check(load().helm_set_knob(name.encode(), int(value)), "helm_set_knob")


def _check(code, where):
    if code != HELM_OK:
        raise HelmError(code, where)


def _stream(stream):
    if stream is not None:
        return ctypes.c_void_p(stream)
    import torch
    if torch.cuda.is_available():
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    return ctypes.c_void_p(0)


_TORCH_DTYPES = {np.dtype(np.complex128): "complex128", np.dtype(np.float64): "float64"}


def _ptr(a, dtype, count=None, out=False):
    """Raw pointer of a torch tensor (device or host) or numpy array (host) of
    `dtype` (complex128 or float64) holding at least `count` elements.  Inputs
    given as numpy arrays of another dtype are converted (a copy); outputs and
    torch tensors must already have the right dtype, be contiguous and large
    enough -- the C ABI would otherwise read or write outside the buffer.
    Returns (pointer, keepalive)."""
    want = np.dtype(dtype)
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.dtype != getattr(torch, _TORCH_DTYPES[want]):
                raise ValueError(f"tensor dtype {a.dtype}, expected torch.{_TORCH_DTYPES[want]}")
            if not a.is_contiguous():
                raise ValueError("tensor must be contiguous")
            if a.device.type not in ("cuda", "cpu"):
                raise ValueError(f"tensor on unsupported device {a.device}")
            if count is not None and a.numel() < count:
                raise ValueError(f"tensor has {a.numel()} elements, need {count}")
            return ctypes.c_void_p(a.data_ptr()), a
    except ImportError:
        pass
    if out:
        if not isinstance(a, np.ndarray) or a.dtype != want or not a.flags["C_CONTIGUOUS"]:
            raise ValueError(f"output must be a contiguous {want} numpy array or torch tensor")
        arr = a
    else:
        arr = np.ascontiguousarray(a, dtype=want)
    if count is not None and arr.size < count:
        raise ValueError(f"array has {arr.size} elements, need {count}")
    return ctypes.c_void_p(arr.ctypes.data), arr


class Problem:
    """helm_assemble: the P1 matrix of Eq. 1a-1b on the '/' mesh (device);
    disc="fd5": helm_assemble_fd5, the paper's five-point scheme (c = 1)."""

    def __init__(self, nx, ny, h, omega, c=None, stream=None, disc="p1"):
        L = load()
        self._keep = []
        cp = ctypes.c_void_p(0)
        if c is not None:
            cp, keep = _ptr(c, np.float64, (nx + 1) * (ny + 1))
            self._keep.append(keep)
        desc = _GridDesc(nx, ny, h, omega, cp)
        handle = ctypes.c_void_p()
        if disc not in ("p1", "fd5"):
            raise ValueError(f"unknown discretisation {disc!r}")
        fn = L.helm_assemble_fd5 if disc == "fd5" else L.helm_assemble
        _check(fn(ctypes.byref(desc), _stream(stream), ctypes.byref(handle)), fn.__name__)
        self.disc = disc
        self.handle = handle
        self.nx, self.ny, self.h, self.omega = nx, ny, h, omega
        self.n = (nx + 1) * (ny + 1)

    @classmethod
    def from_config(cls, cfg, stream=None):
        return cls(cfg.nx, cfg.ny, cfg.h, cfg.omega, np.ascontiguousarray(cfg.c.ravel()), stream)

    def diagonals(self, out, stream=None):
        p, keep = _ptr(out, np.complex128, 4 * self.n, out=True)
        _check(load().helm_get_diagonals(self.handle, p, _stream(stream)), "helm_get_diagonals")
        return keep

    def load_vector(self, f, b, stream=None):
        fp, k1 = _ptr(f, np.complex128, self.n)
        bp, k2 = _ptr(b, np.complex128, self.n, out=True)
        _check(load().helm_load_vector(self.handle, fp, bp, _stream(stream)), "helm_load_vector")
        return k2

    def spmv(self, X, Y, ncols=1, stream=None):
        xp, k1 = _ptr(X, np.complex128, self.n * ncols)
        yp, k2 = _ptr(Y, np.complex128, self.n * ncols, out=True)
        _check(load().helm_spmv(self.handle, xp, yp, ncols, _stream(stream)), "helm_spmv")
        return k2

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _lib is not None:
                _lib.helm_problem_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


@dataclass
class SweepInfo:
    n_strips: int
    nc: int
    wmax: int
    n_segments: int
    solves_per_apply: int
    factor_bytes: int
    model_bytes_per_apply: int
    axis: int
    order: int
    is_double: int


class Sweep:
    """sweep_setup: one directional sweep preconditioner, factored on the device."""

    def __init__(self, problem: Problem, name_or_axis, order=None, n_strips=4, overlap=1, is_double=None,
                 gather=0, n_segments=0, stream=None):
        if isinstance(name_or_axis, str):
            axis, order_, dbl = DIRECTIONS[name_or_axis]
            order = order_
            is_double = dbl if is_double is None else is_double
            self.name = name_or_axis
        else:
            axis = name_or_axis
            is_double = 1 if is_double is None else is_double
            self.name = f"axis{axis}order{order}"
        handle = ctypes.c_void_p()
        _check(load().sweep_setup(problem.handle, axis, order, n_strips, overlap, int(is_double), gather,
                                  n_segments, _stream(stream), ctypes.byref(handle)), "sweep_setup")
        self.handle = handle
        self.problem = problem

    def set_precision(self, separator_bits: int):
        """sweep_set_precision: 32 = opt-in inexact (complex64) separator solve, 64 = exact."""
        _check(load().sweep_set_precision(self.handle, int(separator_bits)), "sweep_set_precision")
        return self

    def info(self) -> SweepInfo:
        arr = (ctypes.c_long * 10)()
        _check(load().sweep_info(self.handle, arr), "sweep_info")
        return SweepInfo(*[int(v) for v in arr])

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _lib is not None:
                _lib.sweep_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


_AXIS = {name: ax for name, (ax, _o, _d) in DIRECTIONS.items()}


def make_sweeps(problem, names, n_strips=4, overlap=1, streams=None, **kw):
    """sweep_setup for several directions, the two axes concurrently: the
    directions of one axis share a factor set and are set up in order on one
    stream, each axis on its own stream and host thread (the library call
    releases the GIL; sweep_setup synchronises its own stream before
    returning).  `streams` maps axis -> CUDA stream handle (default: two
    torch streams).  Returns the Sweep handles in the order of `names`."""
    import threading
    groups = {}
    for k, nm in enumerate(names):
        groups.setdefault(_AXIS[nm], []).append((k, nm))
    if streams is None:
        import torch
        streams = {ax: torch.cuda.Stream().cuda_stream for ax in groups}
    out = [None] * len(names)
    errors = []

    def run(ax):
        try:
            for k, nm in groups[ax]:
                out[k] = Sweep(problem, nm, n_strips=n_strips, overlap=overlap, stream=streams[ax], **kw)
        except Exception as e:  # re-raised in the caller's thread
            errors.append(e)

    threads = [threading.Thread(target=run, args=(ax,)) for ax in groups]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        raise errors[0]
    return out


def _dir_array(dirs):
    arr = (ctypes.c_void_p * len(dirs))()
    for k, d in enumerate(dirs):
        arr[k] = d.handle.value
    return arr


def sweep_apply(dirs, R, Z, ldr=None, ldz=None, stream=None):
    """Z[:, d] = M_d^{-1} R[:, d] for all directions in one launch (ldr = 0
    broadcasts a single vector).  R, Z: (t, n) complex128 row-stacked columns."""
    n = dirs[0].problem.n
    t = len(dirs)
    if ldr is None:
        ldr = 0 if (hasattr(R, "ndim") and R.ndim == 1) else n
    if ldz is None:
        ldz = n
    rp, k1 = _ptr(R, np.complex128, n if ldr == 0 else (t - 1) * ldr + n)
    zp, k2 = _ptr(Z, np.complex128, (t - 1) * ldz + n, out=True)
    _check(load().sweep_apply(_dir_array(dirs), t, rp, ldr, zp, ldz, _stream(stream)), "sweep_apply")
    return k2


def mpgmres_solve(problem, dirs, b, x, tol=1e-6, maxit=200, stream=None, raise_on_noconv=False):
    """Selective MPGMRES on the device; returns (x, stats dict)."""
    hist = (ctypes.c_double * maxit)()
    st = MPGMRESStats()
    st.history = ctypes.cast(hist, ctypes.POINTER(ctypes.c_double))
    st.history_cap = maxit
    n = problem.n
    bp, k1 = _ptr(b, np.complex128, n)
    xp, k2 = _ptr(x, np.complex128, n, out=True)
    code = load().mpgmres_solve(problem.handle, _dir_array(dirs), len(dirs), bp, xp, tol, maxit,
                                ctypes.byref(st), _stream(stream))
    if code not in (HELM_OK, 6, 7) or (raise_on_noconv and code != HELM_OK):
        _check(code, "mpgmres_solve")
    stats = {f: getattr(st, f) for f, _ in MPGMRESStats._fields_ if f != "history"}
    stats["history"] = [hist[i] for i in range(st.iterations)]
    stats["status"] = STATUS.get(code, code)
    return k2, stats


# ---------------------------------------------------------------- direction-parallel solve

def partition_directions(names, nranks):
    """Direction-parallel split: rank r owns the t / nranks
    consecutive global directions r*t_local .. (r+1)*t_local - 1.  t must be a
    multiple of nranks."""
    t = len(names)
    if nranks < 1 or t % nranks:
        raise ValueError(f"{t} directions do not split over {nranks} ranks")
    tl = t // nranks
    return [list(names[r * tl:(r + 1) * tl]) for r in range(nranks)]


class _Bytes:
    """__cuda_array_interface__ / __array_interface__ view of raw bytes."""

    def __init__(self, ptr, nbytes, device):
        iface = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False), "version": 3}
        if device:
            iface["strides"] = None
            iface["stream"] = None
            self.__cuda_array_interface__ = iface
        else:
            self.__array_interface__ = iface


def torch_allgather(group=None, device=True):
    """An all-gather callback (helm_allgather_fn) over torch.distributed: NCCL
    all_gather_into_tensor on the library's stream for device buffers (device
    = True), or a gloo all_gather on host buffers (device = False, CPU tests).
    Keep the returned object alive for the duration of the solve."""
    import torch
    import torch.distributed as dist

    def cb(ctx, send, recv, nbytes, stream):
        try:
            ws = dist.get_world_size(group)
            if device:
                s = torch.as_tensor(_Bytes(send, nbytes, True), device="cuda")
                r = torch.as_tensor(_Bytes(recv, nbytes * ws, True), device="cuda")
                with torch.cuda.stream(torch.cuda.ExternalStream(int(stream or 0))):
                    dist.all_gather_into_tensor(r, s, group=group)
            else:
                s = torch.from_numpy(np.asarray(_Bytes(send, nbytes, False))).clone()
                r = torch.from_numpy(np.asarray(_Bytes(recv, nbytes * ws, False)))
                parts = [torch.empty_like(s) for _ in range(ws)]
                dist.all_gather(parts, s, group=group)
                r.copy_(torch.cat(parts))
            return 0
        except Exception:  # reported to the library as a failed collective
            import traceback
            traceback.print_exc()
            return 1

    return ALLGATHER_FN(cb)


def mpgmres_solve_dist(problem, local_dirs, nranks, rank, b, x, allgather, tol=1e-6, maxit=200, stream=None):
    """mpgmres_solve_dist: this rank's directions local_dirs (global directions
    rank*t_local ..), the new Z / W columns all-gathered by `allgather` (an
    ALLGATHER_FN, e.g. torch_allgather()).  Returns (x, stats dict)."""
    hist = (ctypes.c_double * maxit)()
    st = MPGMRESStats()
    st.history = ctypes.cast(hist, ctypes.POINTER(ctypes.c_double))
    st.history_cap = maxit
    n = problem.n
    bp, k1 = _ptr(b, np.complex128, n)
    xp, k2 = _ptr(x, np.complex128, n, out=True)
    code = load().mpgmres_solve_dist(problem.handle, _dir_array(local_dirs), len(local_dirs), nranks, rank,
                                     allgather, None, bp, xp, tol, maxit, ctypes.byref(st), _stream(stream))
    if code not in (HELM_OK, 6, 7):
        _check(code, "mpgmres_solve_dist")
    stats = {f: getattr(st, f) for f, _ in MPGMRESStats._fields_ if f != "history"}
    stats["history"] = [hist[i] for i in range(st.iterations)]
    stats["status"] = STATUS.get(code, code)
    return k2, stats
