"""Green, Jacobi and Green-Jacobi preconditioners on the device
(preconditioners.py:22-171 of the reference).

``GreenOperator.blocks`` and ``JacobiDiagonal.inv_sqrt`` are host views
downloaded lazily from the device (the reference's tests read them,
test_preconditioners.py:27,32,137,144).
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .operators import _module_of, grid_dim, grid_handle, new_vector, op_handle

PRECONDITIONER_KINDS = ("none", "green", "jacobi", "green-jacobi")
#: eigenvalue cutoff of the pseudo-inverse (preconditioners.py:26); applied
#: on the device in spectral.cu herm_pinv
_EIG_CUTOFF = 1e-12


class GreenOperator:
    """Per-frequency pseudo-inverse blocks of the reference operator
    (preconditioners.py:29-35), resident on the device."""

    def __init__(self, grid, material_ref, handle: N.GreenHandle):
        self.grid = grid
        self.material_ref = material_ref
        self.handle = handle
        self._blocks = None

    @property
    def blocks(self) -> np.ndarray:
        """(n, ..., n//2 + 1, d, d) complex128, Hermitian PSD."""
        if self._blocks is None:
            d = grid_dim(self.grid)
            n = self.grid.n
            shape = (n,) * (d - 1) + (n // 2 + 1, d, d)
            out = np.empty(shape, dtype=np.complex128)
            N.check(N.load().jfftb_green_export_blocks(self.handle.ptr, N.vptr(out)))
            self._blocks = out
        return self._blocks


class JacobiDiagonal:
    """Reciprocal square roots of diag(K), zeros replaced by one
    (preconditioners.py:38-47), resident on the device."""

    def __init__(self, grid, handle: N.JacobiHandle):
        self.grid = grid
        self.handle = handle
        self._inv_sqrt = None

    @property
    def inv_sqrt(self) -> np.ndarray:
        if self._inv_sqrt is None:
            d = grid_dim(self.grid)
            out = np.empty((d,) + (self.grid.n,) * d)
            N.check(N.load().jfftb_jacobi_export(self.handle.ptr, N.vptr(out), N.HOST))
            self._inv_sqrt = out
        return self._inv_sqrt


def assemble_green(grid, material_ref) -> GreenOperator:
    """preconditioners.py:50-80 (impulse responses of K_ref -> spectrum ->
    Hermitised eigen pseudo-inverse with cutoff, DC block zero)."""
    lam, mu = float(material_ref.lambda0), float(material_ref.mu0)
    if mu <= 0.0 or lam + mu <= 0.0:
        raise ValueError(f"stiffness not positive definite (lambda={lam}, mu={mu})")
    return GreenOperator(grid, material_ref, N.GreenHandle(grid_handle(grid), lam, mu))


def green_handle(green) -> N.GreenHandle:
    """Device Green operator of any GreenOperator-like object: ours carry
    one; a reference GreenOperator (built by its own assemble_green) is
    re-assembled on the device from its reference material (cached on it)."""
    h = getattr(green, "handle", None)
    if isinstance(h, N.GreenHandle):
        return h
    h = getattr(green, "_jfftb_green", None)
    if h is None:
        m = green.material_ref
        h = N.GreenHandle(grid_handle(green.grid), float(m.lambda0), float(m.mu0))
        object.__setattr__(green, "_jfftb_green", h)
    return h


def jacobi_handle(jacobi) -> N.JacobiHandle:
    """Device diagonal of any JacobiDiagonal-like object: ours carry one; a
    caller-built one (reference container, e.g. test_preconditioners.py
    unit-diagonal cases) is uploaded from its ``inv_sqrt`` (cached on it)."""
    h = getattr(jacobi, "handle", None)
    if isinstance(h, N.JacobiHandle):
        return h
    arr = jacobi.inv_sqrt
    key = (id(arr), arr.__array_interface__["data"][0])
    c = getattr(jacobi, "_jfftb_jacobi", None)
    if c is None or c[1] != key:
        c = (N.JacobiHandle(None, grid_handle(jacobi.grid), arr), key)
        object.__setattr__(jacobi, "_jfftb_jacobi", c)
    return c[0]


def _apply(kind_code, green, jacobi, r):
    grid = r.grid
    if green is not None and green.grid != grid:
        raise ValueError("residual lives on a different grid")
    if jacobi is not None and jacobi.grid != grid:
        raise ValueError("residual lives on a different grid")
    vals = np.ascontiguousarray(r.values, dtype=np.float64)
    out = np.empty_like(vals)
    gh = green_handle(green).ptr if green is not None else None
    jh = jacobi_handle(jacobi).ptr if jacobi is not None else None
    N.check(N.load().jfftb_apply_precond(kind_code, gh, jh, N.vptr(vals), N.vptr(out), N.HOST))
    return new_vector(r, grid, out)


def apply_green(green: GreenOperator, r):
    """preconditioners.py:83-94: irfftn(G^ . rfftn(r))."""
    if r.grid != green.grid:
        raise ValueError("residual lives on a different grid")
    return _apply(N.PC_GREEN, green, None, r)


def assemble_jacobi(op) -> JacobiDiagonal:
    """preconditioners.py:97-119: d * 2^d comb probes of K on the device."""
    grid = op.grid
    if grid.n % 2 != 0:
        raise ValueError("diagonal probing requires an even node count")
    return JacobiDiagonal(grid, N.JacobiHandle(op_handle(op)))


def apply_jacobi_half(jacobi: JacobiDiagonal, r):
    """preconditioners.py:122-124."""
    return _apply(N.PC_HALF, None, jacobi, r)


def apply_jacobi(jacobi: JacobiDiagonal, r):
    """preconditioners.py:127-129: inv_sqrt * (inv_sqrt * r)."""
    return _apply(N.PC_JACOBI, None, jacobi, r)


def apply_green_jacobi(jacobi: JacobiDiagonal, green: GreenOperator, r):
    """preconditioners.py:132-136: D^-1/2 G D^-1/2 r."""
    return _apply(N.PC_GREEN_JACOBI, green, jacobi, r)


class Preconditioner:
    """Tagged preconditioner variant (preconditioners.py:139-163)."""

    __slots__ = ("kind", "green", "jacobi")

    def __init__(self, kind: str, green=None, jacobi=None):
        if kind not in PRECONDITIONER_KINDS:
            raise ValueError(f"unknown preconditioner {kind!r}; "
                             f"choose one of {PRECONDITIONER_KINDS}")
        if kind in ("green", "green-jacobi") and green is None:
            raise ValueError(f"{kind!r} needs an assembled Green operator")
        if kind in ("jacobi", "green-jacobi") and jacobi is None:
            raise ValueError(f"{kind!r} needs an assembled Jacobi diagonal")
        self.kind, self.green, self.jacobi = kind, green, jacobi

    def __repr__(self):
        return f"Preconditioner(kind={self.kind!r})"

    def apply(self, r):
        if self.kind == "none":
            return new_vector(r, r.grid, r.values.copy())
        if self.kind == "green":
            return apply_green(self.green, r)
        if self.kind == "jacobi":
            return apply_jacobi(self.jacobi, r)
        return apply_green_jacobi(self.jacobi, self.green, r)


def build_preconditioner(kind: str, op, green) -> Preconditioner:
    """preconditioners.py:166-171."""
    jacobi = assemble_jacobi(op) if kind in ("jacobi", "green-jacobi") else None
    used_green = green if kind in ("green", "green-jacobi") else None
    return Preconditioner(kind, green=used_green, jacobi=jacobi)


__all__ = ["PRECONDITIONER_KINDS", "GreenOperator", "JacobiDiagonal", "assemble_green",
           "apply_green", "assemble_jacobi", "apply_jacobi_half", "apply_jacobi",
           "apply_green_jacobi", "Preconditioner", "build_preconditioner", "_module_of"]
