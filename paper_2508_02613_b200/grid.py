"""Periodic regular-grid containers and Mandel algebra, d = 2 or 3.

Mirrors the reference's grid module (/root/reference/pkg/src/jfft/grid.py):
same class names, constructor signatures, validation errors and layouts, but
dimension-generic so 3-D grids use the same API.

Layouts (host, float64, C order, last index contiguous):

* ``ScalarField.values``  ``(n1, ..., nd)``          (grid.py:106-126)
* ``VectorField.values``  ``(d, n1, ..., nd)``       (grid.py:129-145)
* ``QuadField.values``    ``(M, d!, n1, ..., nd)``   (grid.py:148-165)
  with M = 3 (2-D) or 6 (3-D) Mandel components and one quadrature point per
  simplex (2 triangles per pixel, 6 Kuhn tetrahedra per voxel).

The spectrum of a vector field is the real-to-complex half spectrum
``(d, n1, ..., n_{d-1}, nd//2 + 1)`` complex128 (grid.py:195-197):
unnormalised forward transform, ``1/N`` on the inverse.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SQRT2 = float(np.sqrt(2.0))


def mandel_dim(d: int) -> int:
    return 3 if d == 2 else 6


#: Mandel dimension of the 2-D reference (grid.py:28).
MANDEL_DIM = 3


def mandel_pairs(d: int):
    if d == 2:
        return [(0, 0), (1, 1), (0, 1)]
    if d == 3:
        return [(0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1)]
    raise ValueError(f"unsupported dimension d={d}")


def mandel_index(d: int, i: int, j: int) -> int:
    for m, (a, b) in enumerate(mandel_pairs(d)):
        if (a, b) in ((i, j), (j, i)):
            return m
    raise KeyError((i, j))


@dataclass(frozen=True)
class Grid:
    """Regular periodic grid with ``n`` nodes (= pixels/voxels) per direction
    (grid.py:34-78).  ``lengths`` has one entry per dimension; ``d`` follows
    from it (2 unless three lengths are given)."""

    n: int
    lengths: tuple = (1.0, 1.0)

    @property
    def d(self) -> int:
        return len(self.lengths)

    @property
    def shape(self) -> tuple:
        return (self.n,) * self.d

    @property
    def pixel_size(self) -> tuple:
        return tuple(l / self.n for l in self.lengths)

    @property
    def n_nodes(self) -> int:
        return self.n ** self.d

    @property
    def n_pixels(self) -> int:
        return self.n ** self.d

    @property
    def n_simplices(self) -> int:
        return math.factorial(self.d)

    @property
    def n_quad(self) -> int:
        return self.n_simplices * self.n ** self.d

    @property
    def cell_volume(self) -> float:
        return float(np.prod(self.lengths))

    def node_index(self, *idx) -> int:
        """Linear node index with periodic wrap, ``i1`` fastest (grid.py:66-68)."""
        out, stride = 0, 1
        for i in idx:
            out += (i % self.n) * stride
            stride *= self.n
        return out

    def node_coords(self, index: int) -> tuple:
        out = []
        for _ in range(self.d):
            out.append(index % self.n)
            index //= self.n
        return tuple(out)

    pixel_index = node_index
    pixel_coords = node_coords

    def quad_index(self, pixel: int, simplex: int) -> int:
        return simplex * self.n_pixels + pixel


def make_grid(n: int, lengths=(1.0, 1.0)) -> Grid:
    """Validated grid (grid.py:81-96); ``len(lengths)`` selects d = 2 or 3."""
    if int(n) != n or n < 2:
        raise ValueError(f"grid needs n >= 2 nodes per direction, got {n}")
    ls = tuple(float(l) for l in lengths)
    if len(ls) not in (2, 3):
        raise ValueError(f"only d = 2 and d = 3 are supported, got lengths {lengths}")
    if any(l <= 0.0 for l in ls):
        raise ValueError(f"cell side lengths must be positive, got {lengths}")
    return Grid(int(n), ls)


def _as_float_array(values, shape, what: str) -> np.ndarray:
    arr = np.ascontiguousarray(values, dtype=np.float64)
    if arr.shape != shape:
        raise ValueError(f"{what} has shape {arr.shape}, expected {shape}")
    return arr


@dataclass
class ScalarField:
    """One value per pixel (densities) or node (grid.py:106-126)."""

    grid: Grid
    values: np.ndarray
    site: str = "pixel"

    def __post_init__(self):
        if self.site not in ("pixel", "node"):
            raise ValueError(f"unknown site kind {self.site!r}")
        self.values = _as_float_array(self.values, self.grid.shape, "scalar field")

    @classmethod
    def zeros(cls, grid: Grid, site: str = "pixel") -> "ScalarField":
        return cls(grid, np.zeros(grid.shape), site)

    @classmethod
    def full(cls, grid: Grid, value: float, site: str = "pixel") -> "ScalarField":
        return cls(grid, np.full(grid.shape, float(value)), site)


@dataclass
class VectorField:
    """Nodal displacement-like field, one plane per component (grid.py:129-145)."""

    grid: Grid
    values: np.ndarray

    def __post_init__(self):
        self.values = _as_float_array(self.values, (self.grid.d,) + self.grid.shape,
                                      "vector field")

    @classmethod
    def zeros(cls, grid: Grid) -> "VectorField":
        return cls(grid, np.zeros((grid.d,) + grid.shape))

    def component_means(self) -> np.ndarray:
        return self.values.mean(axis=tuple(range(1, self.grid.d + 1)))


@dataclass
class QuadField:
    """Mandel field at quadrature points, ``(M, d!, n, ...)`` (grid.py:148-165)."""

    grid: Grid
    values: np.ndarray

    def __post_init__(self):
        g = self.grid
        self.values = _as_float_array(
            self.values, (mandel_dim(g.d), g.n_simplices) + g.shape, "quadrature field")

    @classmethod
    def zeros(cls, grid: Grid) -> "QuadField":
        return cls(grid, np.zeros((mandel_dim(grid.d), grid.n_simplices) + grid.shape))


def to_mandel(tensor) -> np.ndarray:
    """Symmetric d x d tensor -> Mandel vector (grid.py:172-181)."""
    t = np.asarray(tensor, dtype=np.float64)
    if t.ndim != 2 or t.shape[0] != t.shape[1] or t.shape[0] not in (2, 3):
        raise ValueError(f"expected a 2x2 or 3x3 tensor, got shape {t.shape}")
    if not np.allclose(t, t.T, rtol=0.0, atol=1e-14 * max(1.0, abs(t).max())):
        raise ValueError("tensor is not symmetric")
    d = t.shape[0]
    return np.array([t[i, j] if i == j else SQRT2 * t[i, j] for i, j in mandel_pairs(d)])


def from_mandel(vec) -> np.ndarray:
    """Inverse of :func:`to_mandel` (grid.py:184-188)."""
    v = np.asarray(vec, dtype=np.float64)
    if v.shape not in ((3,), (6,)):
        raise ValueError(f"expected a length-3 or length-6 Mandel vector, got {v.shape}")
    d = 2 if v.shape == (3,) else 3
    t = np.zeros((d, d))
    for m, (i, j) in enumerate(mandel_pairs(d)):
        if i == j:
            t[i, i] = v[m]
        else:
            t[i, j] = t[j, i] = v[m] / SQRT2
    return t


def spectral_shape(grid: Grid) -> tuple:
    """Half-spectrum shape of a vector field (grid.py:195-197)."""
    return (grid.d,) + (grid.n,) * (grid.d - 1) + (grid.n // 2 + 1,)
