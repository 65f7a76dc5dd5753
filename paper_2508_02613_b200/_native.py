"""ctypes binding of libjfftb200.so (include/jfftb200.h).

The library is loaded on first use, never at import time, so that the
reference's fork-based worker pools (experiments.py:326-330) never inherit a
CUDA context.  There is no fallback: if the library is missing or has no GPU
to run on, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("JFFTB_LIB") or os.path.join(HERE, "libjfftb200.so")

OK, EINVAL, ENONFINITE, ECURVATURE, ECUDA = 0, 1, 2, 3, 4
HOST, DEVICE = 0, 1
PC_HALF, PC_NONE, PC_GREEN, PC_JACOBI, PC_GREEN_JACOBI = -1, 0, 1, 2, 3
KIND_CODES = {"none": PC_NONE, "green": PC_GREEN, "jacobi": PC_JACOBI,
              "green-jacobi": PC_GREEN_JACOBI}
CONVERGED_CODE, CAP_CODE = 0, 1

_lock = threading.Lock()
_lib = None
_lib_pid = None


class SolverAbortError(RuntimeError):
    """The PCG recurrence produced a non-finite or non-positive quantity
    (solver.py:40-41)."""


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_SIGS = {
    "jfftb_last_error": (C.c_char_p, []),
    "jfftb_version": (C.c_int, []),
    "jfftb_launch_count": (C.c_int64, [C.c_int]),
    "jfftb_grid_create": (C.c_int, [C.c_int, _I64, _D, C.c_int, C.POINTER(_P)]),
    "jfftb_grid_destroy": (C.c_int, [_P]),
    "jfftb_grid_set_stream": (C.c_int, [_P, _P]),
    "jfftb_grid_synchronize": (C.c_int, [_P]),
    "jfftb_fft_forward": (C.c_int, [_P, _P, _P, C.c_int]),
    "jfftb_fft_inverse": (C.c_int, [_P, _P, _P, C.c_int]),
    "jfftb_op_create": (C.c_int, [_P, _P, C.c_int, C.c_double, C.c_double, C.POINTER(_P)]),
    "jfftb_op_destroy": (C.c_int, [_P]),
    "jfftb_apply_system": (C.c_int, [_P, _P, _P, C.c_int]),
    "jfftb_assemble_rhs": (C.c_int, [_P, _D, _P, C.c_int]),
    "jfftb_total_strain": (C.c_int, [_P, _P, _D, _P, C.c_int]),
    "jfftb_residual_force": (C.c_int, [_P, _P, _D, _P, C.c_int]),
    "jfftb_homogenized_stress": (C.c_int, [_P, _P, _D, _D, C.c_int]),
    "jfftb_green_create": (C.c_int, [_P, C.c_double, C.c_double, C.POINTER(_P)]),
    "jfftb_green_destroy": (C.c_int, [_P]),
    "jfftb_green_export_blocks": (C.c_int, [_P, _P]),
    "jfftb_apply_green": (C.c_int, [_P, _P, _P, C.c_int]),
    "jfftb_jacobi_create": (C.c_int, [_P, C.POINTER(_P)]),
    "jfftb_jacobi_destroy": (C.c_int, [_P]),
    "jfftb_jacobi_from_array": (C.c_int, [_P, _P, C.c_int, C.POINTER(_P)]),
    "jfftb_jacobi_export": (C.c_int, [_P, _P, C.c_int]),
    "jfftb_apply_precond": (C.c_int, [C.c_int, _P, _P, _P, _P, C.c_int]),
    "jfftb_pcg": (C.c_int, [_P, C.c_int, _P, _P, _P, _P, C.c_int, C.c_double, C.c_int, _P,
                            _D, C.POINTER(C.c_int), C.POINTER(C.c_int), _D]),
    "jfftb_profile_start": (C.c_int, [_P]),
    "jfftb_profile_read": (C.c_int, [_P, _D, _I64, C.c_int]),
    "jfftb_debug_fused_apply": (C.c_int, [_P, _P, C.c_int, _P, _P]),
    "jfftb_binomial_filter": (C.c_int, [_P, _P, C.c_int, C.c_int]),
    "jfftb_field_minmax": (C.c_int, [_P, _P, _D, C.c_int]),
    "jfftb_rescale_contrast": (C.c_int, [_P, _P, C.c_double, C.c_int]),
    "jfftb_threshold": (C.c_int, [_P, _P, C.c_double, C.c_int]),
    "jfftb_simp_projection": (C.c_int, [_P, _P, C.c_double, C.c_double, C.c_int]),
    "jfftb_field_layout": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.c_int]),
    "jfftb_load_pairings": (C.c_int, [_P, C.c_int, _P, _D, _D, _D, _P, C.c_int]),
    "jfftb_pcg_batch": (C.c_int, [_P, C.c_int, _P, _P, _P, C.c_int, _P, C.c_int, C.c_double,
                                  C.c_int, _P, _D, C.POINTER(C.c_int), C.POINTER(C.c_int), _D]),
    "jfftb_comm_unique_id": (C.c_int, [C.c_char_p]),
    "jfftb_comm_create_nccl": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    "jfftb_comm_create_local": (C.c_int, [C.c_int, C.c_int, C.POINTER(_P)]),
    "jfftb_comm_destroy": (C.c_int, [_P]),
    "jfftb_dist_create": (C.c_int, [_P, _I64, _D, _P, C.c_int, C.c_double, C.c_double,
                                    C.c_double, C.c_double, C.c_int, C.POINTER(_P)]),
    "jfftb_dist_destroy": (C.c_int, [_P]),
    "jfftb_dist_assemble_rhs": (C.c_int, [_P, _D, _P, C.c_int]),
    "jfftb_dist_jacobi_export": (C.c_int, [_P, _P, C.c_int]),
    "jfftb_dist_pcg": (C.c_int, [_P, _P, C.c_int, C.c_double, C.c_int, _P, _D,
                                 C.POINTER(C.c_int), C.POINTER(C.c_int), _D]),
    "jfftb_dist_info": (C.c_int, [_P, _I64]),
}
EXPORTED = tuple(_SIGS)


def load(path: str = LIB_PATH):
    """Load (once per process) and type the C ABI."""
    global _lib, _lib_pid
    with _lock:
        if _lib is not None and _lib_pid == os.getpid():
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: the CUDA path has no fallback; build it with "
                "`python -m paper_2508_02613_b200.build`")
        lib = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib, _lib_pid = lib, os.getpid()
        return lib


def last_error() -> str:
    msg = load().jfftb_last_error()
    return msg.decode() if msg else ""


def check(status: int, abort_cls=None):
    if status == OK:
        return
    msg = last_error()
    if status == EINVAL:
        raise ValueError(msg)
    if status in (ENONFINITE, ECURVATURE):
        raise (abort_cls or SolverAbortError)(msg)
    raise RuntimeError(f"libjfftb200: {msg}")


def dptr(a: np.ndarray):
    """Pointer to a C-contiguous float64 host array."""
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def vptr(a: np.ndarray):
    assert a.flags.c_contiguous
    return C.c_void_p(a.ctypes.data)


def device_id() -> int:
    return int(os.environ.get("JFFTB_DEVICE", "0"))


# ---------------------------------------------------------------------------
# handles
# ---------------------------------------------------------------------------

class _Handle:
    _destroy = None

    def __init__(self, ptr):
        self.ptr = ptr
        self._pid = os.getpid()

    def __del__(self):
        try:
            if self.ptr and self._pid == os.getpid() and _lib is not None:
                getattr(_lib, self._destroy)(self.ptr)
        except Exception:
            pass
        self.ptr = None


class GridHandle(_Handle):
    _destroy = "jfftb_grid_destroy"

    def __init__(self, d, n, lengths, device=None):
        lib = load()
        ns = (C.c_int64 * d)(*n)
        ls = (C.c_double * d)(*lengths)
        out = C.c_void_p()
        check(lib.jfftb_grid_create(d, ns, ls, device_id() if device is None else device,
                                    C.byref(out)))
        super().__init__(out)
        self.d, self.n, self.lengths = d, tuple(n), tuple(lengths)
        self.shape = tuple(n)
        self.N = int(np.prod(n))
        self.spec_shape = (d,) + tuple(n[:-1]) + (n[-1] // 2 + 1,)

    def set_stream(self, stream_ptr: int | None):
        """Run on a caller's CUDA stream (e.g. ``torch.cuda.current_stream()
        .cuda_stream``).  Handle 0 -- torch's default stream -- is the legacy
        default stream, passed to the library as cudaStreamLegacy (0x1)."""
        check(load().jfftb_grid_set_stream(self.ptr, C.c_void_p(stream_ptr or 1)))

    def synchronize(self):
        check(load().jfftb_grid_synchronize(self.ptr))

    def profile_start(self):
        check(load().jfftb_profile_start(self.ptr))

    def profile_read(self, stop: bool = True):
        """(stage_ms[8], iterations) accumulated since profile_start."""
        ms = np.zeros(8)
        it = C.c_int64(0)
        check(load().jfftb_profile_read(self.ptr, dptr(ms), C.byref(it), 1 if stop else 0))
        return ms, it.value


class OpHandle(_Handle):
    _destroy = "jfftb_op_destroy"

    def __init__(self, grid: GridHandle, rho, lam, mu, where=HOST):
        out = C.c_void_p()
        ptr = vptr(rho) if where == HOST else C.c_void_p(rho)
        check(load().jfftb_op_create(grid.ptr, ptr, where, float(lam), float(mu), C.byref(out)))
        super().__init__(out)
        self.grid = grid


class GreenHandle(_Handle):
    _destroy = "jfftb_green_destroy"

    def __init__(self, grid: GridHandle, lam, mu):
        out = C.c_void_p()
        check(load().jfftb_green_create(grid.ptr, float(lam), float(mu), C.byref(out)))
        super().__init__(out)
        self.grid = grid


class JacobiHandle(_Handle):
    _destroy = "jfftb_jacobi_destroy"

    def __init__(self, op: OpHandle | None, grid: GridHandle | None = None, inv_sqrt=None):
        """Probed from ``op`` (assemble_jacobi), or, with ``op=None``, uploaded
        from a caller's ``inv_sqrt`` array on ``grid``."""
        out = C.c_void_p()
        if op is not None:
            check(load().jfftb_jacobi_create(op.ptr, C.byref(out)))
        else:
            arr = np.ascontiguousarray(inv_sqrt, dtype=np.float64)
            check(load().jfftb_jacobi_from_array(grid.ptr, vptr(arr), HOST, C.byref(out)))
        super().__init__(out)
        self.op = op
        self.grid = op.grid if op is not None else grid


_grid_cache: dict = {}


def grid_handle(d: int, n, lengths, device: int | None = None) -> GridHandle:
    """One grid context per (d, n, lengths, device) and process; ``device``
    defaults to JFFTB_DEVICE (the containers' device)."""
    dev = device_id() if device is None else int(device)
    key = (os.getpid(), d, tuple(int(k) for k in n), tuple(float(l) for l in lengths), dev)
    h = _grid_cache.get(key)
    if h is None:
        h = GridHandle(d, key[2], key[3], device=dev)
        _grid_cache[key] = h
    return h


def register_grid(h: GridHandle) -> None:
    """Make an explicitly created grid context the one the Python API uses
    for its (d, n, lengths) (e.g. a context bound to a torch stream)."""
    key = (os.getpid(), h.d, tuple(int(k) for k in h.n), tuple(float(l) for l in h.lengths),
           device_id())
    _grid_cache[key] = h


def launch_count(reset: bool = False) -> int:
    return int(load().jfftb_launch_count(1 if reset else 0))
