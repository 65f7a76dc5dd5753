"""Seeded synthetic inputs for the BASELINE.json configurations.

These build the density (= Young's modulus E(x)) fields the benchmark and the
parity tests feed the PCG path.  They are input preparation, not the hot
path.  The 2-D recipe follows SURVEY.md section 8(d): a Bernoulli(0.5) pixel
field, ``i`` passes of the reference's binomial filter
(microstructures.py:73-82 -- BASELINE's "3x3 Gaussian, sigma = 1 px" is read
as that kernel), then ``rescale_contrast`` (microstructures.py:104-115).
The 3-D recipes (spheres, crack discs, SIMP-thresholded noise) are this
build's reading of BASELINE configs 3-5; DESIGN.md records the choices.
"""

from __future__ import annotations

import numpy as np

NU = 0.3


def lame_from_poisson(nu: float = NU):
    """Material for rho := E(x): lambda = nu / ((1+nu)(1-2nu)), mu = 1/(2(1+nu))."""
    return nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), 1.0 / (2.0 * (1.0 + nu))


def binomial_filter(v: np.ndarray) -> np.ndarray:
    """One periodic pass of the separable [1 2 1]/4 kernel along every axis,
    same operation order as microstructures.py:79-81."""
    for ax in range(v.ndim):
        v = (v + np.roll(v, 1, axis=ax) / 2 + np.roll(v, -1, axis=ax) / 2) / 2
    return v


def rescale_contrast(v: np.ndarray, chi: float) -> np.ndarray:
    """Affine map onto [1/chi, 1] (microstructures.py:104-115)."""
    lo, hi = v.min(), v.max()
    if hi <= lo:
        raise ValueError("cannot rescale a constant field to a target contrast")
    soft = 0.0 if np.isinf(chi) else 1.0 / chi
    return soft + (1.0 - soft) * (v - lo) / (hi - lo)


def bernoulli_smoothed(n: int, filters: int, chi: float = 1e4, seed: int = 0,
                       d: int = 2) -> np.ndarray:
    """Configs 1-2: seeded Bernoulli(0.5) -> ``filters`` binomial passes ->
    contrast ``chi`` (E = 1/chi + (1 - 1/chi) phi)."""
    rng = np.random.default_rng(seed)
    v = (rng.random((n,) * d) < 0.5).astype(float)
    for _ in range(filters):
        v = binomial_filter(v)
    return rescale_contrast(v, chi)


def _min_image(delta: np.ndarray, period: float) -> np.ndarray:
    return delta - period * np.round(delta / period)


def random_spheres(n: int = 128, count: int = 32, rmin: float = 6.0,
                   rmax: float = 16.0, filters: int = 5, emin: float = 1e-3,
                   seed: int = 0) -> np.ndarray:
    """Config 3: stiff spheres (phi = 1 inside any sphere, periodic minimum
    image), ``filters`` 3-D binomial passes, min-max rescale,
    E = emin + (1 - emin) phi."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.0, n, (count, 3))
    radii = rng.uniform(rmin, rmax, count)
    ax = np.arange(n, dtype=float) + 0.5
    phi = np.zeros((n, n, n))
    for c, r in zip(centres, radii):
        d0 = _min_image(ax - c[0], n)[:, None, None] ** 2
        d1 = _min_image(ax - c[1], n)[None, :, None] ** 2
        d2 = _min_image(ax - c[2], n)[None, None, :] ** 2
        phi[(d0 + d1 + d2) <= r * r] = 1.0
    for _ in range(filters):
        phi = binomial_filter(phi)
    lo, hi = phi.min(), phi.max()
    phi = (phi - lo) / (hi - lo)
    return emin + (1.0 - emin) * phi


def crack_discs_params(n: int = 512, count: int = 64, rmin: float = 8.0,
                       rmax: float = 32.0, seed: int = 0):
    """Config 4 geometry: disc centres uniform in the cell, normals uniform
    on S^2, radii uniform in [rmin, rmax] (voxel units)."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.0, n, (count, 3))
    normals = rng.normal(size=(count, 3))
    normals /= np.linalg.norm(normals, axis=1, keepdims=True)
    radii = rng.uniform(rmin, rmax, count)
    return centres, normals, radii


def crack_discs(n: int = 512, count: int = 64, ell: float = 4.0,
                emin: float = 1e-4, seed: int = 0, chunk: int = 8) -> np.ndarray:
    """Config 4: phi = exp(-dist/ell) to the nearest disc (periodic minimum
    image per disc), E = (1 - phi)^2 + emin.  CPU version, for the small
    parity grids; bench-size grids use the device generator."""
    centres, normals, radii = crack_discs_params(n, count, seed=seed)
    ax = np.arange(n, dtype=float) + 0.5
    out = np.empty((n, n, n))
    for i0 in range(0, n, chunk):
        x0 = ax[i0:i0 + chunk]
        dmin = np.full((len(x0), n, n), np.inf)
        for c, nr, r in zip(centres, normals, radii):
            v0 = _min_image(x0 - c[0], n)[:, None, None]
            v1 = _min_image(ax - c[1], n)[None, :, None]
            v2 = _min_image(ax - c[2], n)[None, None, :]
            hgt = v0 * nr[0] + v1 * nr[1] + v2 * nr[2]
            rad2 = np.maximum(v0 * v0 + v1 * v1 + v2 * v2 - hgt * hgt, 0.0)
            rad = np.sqrt(rad2)
            dist = np.where(rad <= r, np.abs(hgt),
                            np.sqrt(hgt * hgt + (rad - r) ** 2))
            np.minimum(dmin, dist, out=dmin)
        phi = np.exp(-dmin / ell)
        out[i0:i0 + chunk] = (1.0 - phi) ** 2 + emin
    return out


def crack_discs_device(n=512, count: int = 64, ell: float = 4.0, emin: float = 1e-4,
                       seed: int = 0, device="cuda", out=None, planes=None, rows=None):
    """Device (torch) version of :func:`crack_discs` with the same seeded
    geometry, for bench-size grids.  ``n`` is an int (cubic) or a shape
    (n0, n1, n2); ``planes = (lo, hi)`` generates only those axis-0 planes,
    ``rows = (lo, hi)`` only those axis-1 rows (one slab of a distributed
    run, paper_2508_02613_b200.dist).  Returns a float64 tensor."""
    import torch
    shape = (n,) * 3 if isinstance(n, int) else tuple(int(k) for k in n)
    if isinstance(n, int):
        centres, normals, radii = crack_discs_params(n, count, seed=seed)
    else:
        rng = np.random.default_rng(seed)
        centres = rng.uniform(0.0, 1.0, (count, 3)) * np.array(shape, dtype=float)
        normals = rng.normal(size=(count, 3))
        normals /= np.linalg.norm(normals, axis=1, keepdims=True)
        radii = rng.uniform(8.0, 32.0, count)
    lo, hi = planes if planes is not None else (0, shape[0])
    axes = [torch.arange(k, dtype=torch.float64, device=device) + 0.5 for k in shape]
    n1, n2 = shape[1], shape[2]
    r0, r1 = rows if rows is not None else (0, n1)
    axes[1] = axes[1][r0:r1]
    if out is None:
        out = torch.empty((hi - lo, r1 - r0, n2), dtype=torch.float64, device=device)
    chunk = max(1, min(hi - lo, (1 << 24) // ((r1 - r0) * n2)))
    for i0 in range(lo, hi, chunk):
        x0 = axes[0][i0:min(i0 + chunk, hi)]
        dmin = torch.full((len(x0), r1 - r0, n2), float("inf"), dtype=torch.float64,
                          device=device)
        for c, nr, r in zip(centres, normals, radii):
            v0 = x0 - c[0]
            v0 = (v0 - shape[0] * torch.round(v0 / shape[0]))[:, None, None]
            v1 = axes[1] - c[1]
            v1 = (v1 - n1 * torch.round(v1 / n1))[None, :, None]
            v2 = axes[2] - c[2]
            v2 = (v2 - n2 * torch.round(v2 / n2))[None, None, :]
            hgt = v0 * float(nr[0]) + v1 * float(nr[1]) + v2 * float(nr[2])
            rad = torch.sqrt(torch.clamp(v0 * v0 + v1 * v1 + v2 * v2 - hgt * hgt, min=0.0))
            dist = torch.where(rad <= float(r), hgt.abs(),
                               torch.sqrt(hgt * hgt + (rad - float(r)) ** 2))
            torch.minimum(dmin, dist, out=dmin)
        phi = torch.exp(-dmin / ell)
        out[i0 - lo:i0 - lo + len(x0)] = (1.0 - phi) ** 2 + emin
    return out


def simp_density(n: int = 1024, filters: int = 8, beta: float = 8.0, emin: float = 1e-6,
                 seed: int = 0) -> np.ndarray:
    """Config 5 (host recipe): seeded uniform noise -> ``filters`` 3-D
    binomial passes -> tanh(beta (rho - 1/2)) -> min-max to [0, 1] ->
    SIMP E = emin + rho^3 (contrast ~1e6).  ``generators.simp_density_device``
    runs the same steps in device memory for the 1024^3 grid."""
    rng = np.random.default_rng(seed)
    v = rng.random((n,) * 3)
    for _ in range(filters):
        v = binomial_filter(v)
    v = np.tanh(beta * (v - 0.5))
    lo, hi = v.min(), v.max()
    v = (v - lo) / (hi - lo)
    return emin + v * v * v


def mandel_shear(d: int, i: int, j: int, gamma: float = 0.5) -> np.ndarray:
    """Mandel vector of the symmetric strain with eps_ij = eps_ji = gamma."""
    from .grid import mandel_index
    m = 3 if d == 2 else 6
    e = np.zeros(m)
    e[mandel_index(d, i, j)] = np.sqrt(2.0) * gamma
    return e
