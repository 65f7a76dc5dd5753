"""System operator K(rho) = B^T W C(rho) B on the device (operators.py:15-101).

Same names, signatures, validation and error types as the reference; the
arithmetic runs in libjfftb200.so.  Functions accept the reference's own
containers as well as this package's (anything with ``.grid`` (``n``,
``lengths``) and ``.values``), and return containers of the caller's classes.
"""

from __future__ import annotations

import math
import sys
from dataclasses import dataclass

import numpy as np

from . import _native as N


@dataclass(frozen=True)
class QuadratureWeights:
    """fem.py:24-38: every quadrature point carries prod(h) / d!."""

    grid: object
    per_point: float

    @property
    def total(self) -> float:
        return self.per_point * self.grid.n_quad


def quadrature_weights(grid) -> QuadratureWeights:
    h = grid.pixel_size
    return QuadratureWeights(grid, float(np.prod(h)) / math.factorial(len(h)))


def grid_dim(grid) -> int:
    return len(grid.lengths)


def grid_handle(grid) -> N.GridHandle:
    d = grid_dim(grid)
    return N.grid_handle(d, (grid.n,) * d, grid.lengths)


def _module_of(obj):
    return sys.modules[type(obj).__module__]


def new_vector(like, grid, values):
    return type(like)(grid, values)


def new_quad(like, grid, values):
    return _module_of(like).QuadField(grid, values)


def _vec_values(u, grid) -> np.ndarray:
    if u.grid != grid:
        raise ValueError("displacement lives on a different grid")
    return np.ascontiguousarray(u.values, dtype=np.float64)


@dataclass(frozen=True)
class SystemOperator:
    """operators.py:15-35 -- grid, pixel densities, base material, weights.

    The device copy of the density is created lazily on first use and cached
    on the object (density arrays are treated as immutable, as the reference
    does)."""

    grid: object
    density: object
    material: object
    weights: QuadratureWeights

    def __post_init__(self):
        if self.density.grid != self.grid or self.weights.grid != self.grid:
            raise ValueError("density/weights grid mismatch")
        if self.density.site != "pixel":
            raise ValueError("density must be a pixel field")
        if np.any(self.density.values < 0.0):
            raise ValueError("negative density")


def make_operator(density, material) -> SystemOperator:
    """operators.py:38-40."""
    grid = density.grid
    return SystemOperator(grid, density, material, quadrature_weights(grid))


def op_handle(op) -> N.OpHandle:
    """Device operator for any SystemOperator-like object (cached on it)."""
    h = getattr(op, "_jfftb_op", None)
    rho = op.density.values
    key = (id(rho), rho.__array_interface__["data"][0])
    if h is None or h[1] != key:
        gh = grid_handle(op.grid)
        arr = np.ascontiguousarray(rho, dtype=np.float64)
        handle = N.OpHandle(gh, arr, op.material.lambda0, op.material.mu0)
        h = (handle, key)
        object.__setattr__(op, "_jfftb_op", h)
    return h[0]


def apply_system(op, u):
    """operators.py:51-58: K(rho) u."""
    if u.grid != op.grid:
        raise ValueError("displacement lives on a different grid")
    h = op_handle(op)
    vals = _vec_values(u, op.grid)
    out = np.empty_like(vals)
    N.check(N.load().jfftb_apply_system(h.ptr, N.vptr(vals), N.vptr(out), N.HOST))
    return new_vector(u, op.grid, out)


def _eps_bar(op, eps_bar) -> np.ndarray:
    d = grid_dim(op.grid)
    m = 3 if d == 2 else 6
    e = np.asarray(eps_bar, dtype=np.float64)
    if e.shape != (m,):
        raise ValueError(f"macroscopic strain must have shape ({m},)")
    if not np.all(np.isfinite(e)):
        raise ValueError("macroscopic strain must be finite")
    return np.ascontiguousarray(e)


def _vector_class(op):
    # the VectorField class that belongs with the operator's containers
    return _module_of(op.density).VectorField


def assemble_rhs(op, eps_bar):
    """operators.py:61-76: f = -B^T W rho C0 E."""
    e = _eps_bar(op, eps_bar)
    h = op_handle(op)
    d = grid_dim(op.grid)
    out = np.empty((d,) + (op.grid.n,) * d)
    N.check(N.load().jfftb_assemble_rhs(h.ptr, N.dptr(e), N.vptr(out), N.HOST))
    return _vector_class(op)(op.grid, out)


def total_strain(op, u, eps_bar):
    """operators.py:79-83: E + B u at the quadrature points."""
    e = np.ascontiguousarray(np.asarray(eps_bar, dtype=np.float64))
    d = grid_dim(op.grid)
    if e.shape != ((3 if d == 2 else 6),):
        raise ValueError("macroscopic strain has the wrong shape")
    h = op_handle(op)
    vals = _vec_values(u, op.grid)
    out = np.empty(((3 if d == 2 else 6), math.factorial(d)) + (op.grid.n,) * d)
    N.check(N.load().jfftb_total_strain(h.ptr, N.vptr(vals), N.dptr(e), N.vptr(out), N.HOST))
    return new_quad(u, op.grid, out)


def residual_force(op, u, eps_bar):
    """operators.py:86-95: -B^T W sigma(rho, E + B u)."""
    e = np.ascontiguousarray(np.asarray(eps_bar, dtype=np.float64))
    h = op_handle(op)
    vals = _vec_values(u, op.grid)
    out = np.empty_like(vals)
    N.check(N.load().jfftb_residual_force(h.ptr, N.vptr(vals), N.dptr(e), N.vptr(out), N.HOST))
    return new_vector(u, op.grid, out)


def homogenized_stress(op, u, eps_bar) -> np.ndarray:
    """operators.py:98-101: (w/|Y|) sum_Q rho C0 (E + B u)."""
    e = np.ascontiguousarray(np.asarray(eps_bar, dtype=np.float64))
    d = grid_dim(op.grid)
    if e.shape != ((3 if d == 2 else 6),):
        raise ValueError("macroscopic strain has the wrong shape")
    h = op_handle(op)
    vals = _vec_values(u, op.grid)
    sig = np.empty(3 if d == 2 else 6)
    N.check(N.load().jfftb_homogenized_stress(h.ptr, N.vptr(vals), N.dptr(e), N.dptr(sig),
                                              N.HOST))
    return sig
