"""PCG with Green-norm termination, and the Newton driver, on the device
(solver.py:1-185 of the reference).

The whole recurrence of one ``pcg`` call runs inside libjfftb200.so
(``jfftb_pcg``): one host->device copy of the right-hand side, device-side
alpha/beta/termination, one device->host copy of the solution and history.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .operators import (grid_dim, make_operator, new_vector, op_handle, residual_force)
from .preconditioners import apply_green, assemble_green, build_preconditioner

DEFAULT_ETA_CG = 1e-6
DEFAULT_MAX_ITER = 999
CONVERGED = "converged"
ITERATION_CAP = "iteration-cap"
DEFAULT_LAMBDA0 = 2.0 / 3.0
DEFAULT_MU0 = 0.5

SolverAbortError = N.SolverAbortError


@dataclass
class SolveReport:
    """solver.py:44-57: ``residual_history`` has ``iterations + 1`` entries."""

    iterations: int
    residual_history: list
    terminated: str
    wall_time: float
    solution: object
    newton_steps: int = 0


def pcg(op, rhs, preconditioner, green, eta: float = DEFAULT_ETA_CG,
        max_iter: int = DEFAULT_MAX_ITER, abort_error=None) -> SolveReport:
    """Solve K u = rhs from x0 = 0 (solver.py:64-140).

    Same contract as the reference: absolute termination ``<r, G r> <= eta``
    checked at k = 0 and after every update, ``iterations`` = number of
    search-direction updates, cap reported as ``iteration-cap``, zero-mean
    solution, ``SolverAbortError`` on NaN/Inf or curvature <= 0.
    """
    start = time.perf_counter()
    kind = preconditioner.kind
    code = N.KIND_CODES[kind]
    h = op_handle(op)
    vals = np.ascontiguousarray(rhs.values, dtype=np.float64)
    x = np.empty_like(vals)
    max_iter = int(max_iter)
    hist = np.zeros(max_iter + 1)
    iters = C.c_int(0)
    term = C.c_int(0)
    wall = C.c_double(0.0)
    from .preconditioners import green_handle, jacobi_handle
    gpc = green_handle(preconditioner.green).ptr if preconditioner.green is not None else None
    jac = jacobi_handle(preconditioner.jacobi).ptr if preconditioner.jacobi is not None else None
    status = N.load().jfftb_pcg(h.ptr, code, gpc, jac, green_handle(green).ptr, N.vptr(vals), N.HOST,
                                float(eta), max_iter, N.vptr(x), N.dptr(hist), C.byref(iters),
                                C.byref(term), C.byref(wall))
    N.check(status, abort_error or SolverAbortError)
    it = iters.value
    return SolveReport(it, [float(v) for v in hist[:it + 1]],
                       CONVERGED if term.value == N.CONVERGED_CODE else ITERATION_CAP,
                       time.perf_counter() - start, new_vector(rhs, rhs.grid, x))


def pcg_device(op_h: N.OpHandle, kind: str, green_h: N.GreenHandle, jac_h, rhs_ptr: int,
               x_ptr: int, eta: float, max_iter: int, green_pc_h=None):
    """Device-resident PCG: ``rhs_ptr``/``x_ptr`` are device addresses (e.g.
    ``torch.Tensor.data_ptr()``) on the grid's device and stream.
    Returns (iterations, history, terminated, wall_s)."""
    hist = np.zeros(int(max_iter) + 1)
    iters, term, wall = C.c_int(0), C.c_int(0), C.c_double(0.0)
    gpc = (green_pc_h or green_h).ptr if kind in ("green", "green-jacobi") else None
    jac = jac_h.ptr if (jac_h is not None and kind in ("jacobi", "green-jacobi")) else None
    status = N.load().jfftb_pcg(op_h.ptr, N.KIND_CODES[kind], gpc, jac, green_h.ptr,
                                C.c_void_p(rhs_ptr), N.DEVICE, float(eta), int(max_iter),
                                C.c_void_p(x_ptr), N.dptr(hist), C.byref(iters), C.byref(term),
                                C.byref(wall))
    N.check(status)
    it = iters.value
    return it, hist[:it + 1].tolist(), (CONVERGED if term.value == 0 else ITERATION_CAP), \
        wall.value


def pcg_device_batch(op_h: N.OpHandle, kind: str, green_h: N.GreenHandle, jac_h, nrhs: int,
                     rhs_ptr: int, x_ptr: int, eta: float, max_iter: int, green_pc_h=None):
    """``nrhs`` device-resident solves at once (jfftb_pcg_batch: one launch
    per stage for all of them; fused 3-D grids, green / green-jacobi).
    ``rhs_ptr``/``x_ptr``: nrhs vector fields back to back on the device.
    Returns per solve (iterations, history, terminated) and the wall time."""
    m = int(max_iter) + 1
    hist = np.zeros(nrhs * m)
    iters = (C.c_int * nrhs)()
    terms = (C.c_int * nrhs)()
    wall = C.c_double(0.0)
    gpc = (green_pc_h or green_h).ptr
    jac = jac_h.ptr if (jac_h is not None and kind == "green-jacobi") else None
    status = N.load().jfftb_pcg_batch(op_h.ptr, N.KIND_CODES[kind], gpc, jac, green_h.ptr, nrhs,
                                      C.c_void_p(rhs_ptr), N.DEVICE, float(eta), int(max_iter),
                                      C.c_void_p(x_ptr), N.dptr(hist), iters, terms,
                                      C.byref(wall))
    N.check(status)
    out = [(iters[l], hist[l * m:l * m + iters[l] + 1].tolist(),
            CONVERGED if terms[l] == 0 else ITERATION_CAP) for l in range(nrhs)]
    return out, wall.value


def _dot(a, b) -> float:
    return float(np.vdot(a.values, b.values))


def newton_solve(density, eps_bar, preconditioner: str = "green", material=None,
                 eta: float = DEFAULT_ETA_CG, max_iter: int = DEFAULT_MAX_ITER, green=None,
                 max_newton: int = 10) -> SolveReport:
    """solver.py:143-185: Newton loop around pcg; one step for the linear law."""
    from .material import isotropic_material
    start = time.perf_counter()
    if material is None:
        material = isotropic_material(DEFAULT_LAMBDA0, DEFAULT_MU0, grid_dim(density.grid))
    op = make_operator(density, material)
    if green is None:
        green = assemble_green(op.grid, material)
    precond = build_preconditioner(preconditioner, op, green)
    d = grid_dim(op.grid)
    vec_cls = type(op.density).__module__
    import sys
    VectorField = sys.modules[vec_cls].VectorField
    u = VectorField.zeros(op.grid)
    report = SolveReport(0, [0.0], CONVERGED, 0.0, u)
    steps = 0
    while True:
        force = residual_force(op, u, eps_bar)
        gnorm2 = _dot(force, apply_green(green, force))
        if gnorm2 <= eta or steps >= max_newton:
            if steps == 0:
                report.residual_history = [gnorm2]
                report.terminated = CONVERGED if gnorm2 <= eta else ITERATION_CAP
            break
        report = pcg(op, force, precond, green, eta=eta, max_iter=max_iter)
        u.values += report.solution.values
        steps += 1
        if report.terminated != CONVERGED:
            break
    u.values -= u.values.mean(axis=tuple(range(1, d + 1))).reshape((d,) + (1,) * d)
    report.solution = u
    report.newton_steps = steps
    report.wall_time = time.perf_counter() - start
    return report
