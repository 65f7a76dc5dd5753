"""Isotropic Mandel stiffness (material.py:12-46 of the reference), d = 2 or 3.

Only the Lame constants reach the device: the kernels evaluate
sigma = lambda tr(eps) I + 2 mu eps directly, which is C0 applied in Mandel
form.  ``stiffness`` keeps the reference's 2-D 3x3 matrix; ``stiffness_for``
gives the 6x6 3-D one.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def isotropic_stiffness(d: int, lam: float, mu: float) -> np.ndarray:
    m = 3 if d == 2 else 6
    c = np.zeros((m, m))
    for i in range(d):
        for j in range(d):
            c[i, j] = lam
        c[i, i] = lam + 2.0 * mu
    for k in range(d, m):
        c[k, k] = 2.0 * mu
    return c


@dataclass(frozen=True)
class MaterialModel:
    """Base stiffness of the solid phase; local stiffness is ``rho * C0``."""

    lambda0: float
    mu0: float
    stiffness: np.ndarray = field(repr=False)

    def __post_init__(self):
        object.__setattr__(self, "stiffness", np.asarray(self.stiffness, dtype=np.float64))

    def stiffness_for(self, d: int) -> np.ndarray:
        return isotropic_stiffness(d, self.lambda0, self.mu0)


def isotropic_material(lambda0: float, mu0: float, d: int = 2) -> MaterialModel:
    """material.py:25-46: rejects mu <= 0 or lambda + mu <= 0."""
    lam, mu = float(lambda0), float(mu0)
    if mu <= 0.0 or lam + mu <= 0.0:
        raise ValueError(f"stiffness not positive definite (lambda={lam}, mu={mu})")
    return MaterialModel(lam, mu, isotropic_stiffness(d, lam, mu))
