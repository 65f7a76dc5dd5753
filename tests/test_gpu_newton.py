"""newton_solve + residual_force on the device, mirroring the
reference's Newton certificates /root/reference/pkg/tests/test_solver.py:
105-159 (single step for the linear law, the linearity certificate, zero
load, uniform-medium stress, and the recomputed residual passing the same
Green-norm test), in 2-D and 3-D.

The reference's laminate / cosine densities (microstructures.py:16-51,
118-130) are restated here so the test runs without the reference."""

import numpy as np
import pytest

from oracle import jfft_oracle as X
from paper_2508_02613_b200 import grid as G
from paper_2508_02613_b200.material import isotropic_material
from paper_2508_02613_b200.operators import (apply_system, assemble_rhs, homogenized_stress,
                                             make_operator, residual_force)
from paper_2508_02613_b200.preconditioners import (apply_green, assemble_green,
                                                   build_preconditioner)
from paper_2508_02613_b200.solver import CONVERGED, newton_solve, pcg

pytestmark = pytest.mark.gpu


def _coords(p):
    x = np.arange(p) / p  # microstructures.py:16-18
    return np.meshgrid(x, x, indexing="ij")


def laminate(p, chi):
    """microstructures.py:21-34."""
    x1, _ = _coords(p)
    return chi + (1.0 - chi) / (1.0 - 1.0 / p) * x1


def cosine(p, chi):
    """microstructures.py:37-51 (finite contrast)."""
    x1, x2 = _coords(p)
    return 0.5 + 0.25 * (np.cos(2.0 * np.pi * (x1 - x2)) + np.cos(2.0 * np.pi * (x2 + x1))) + 1.0 / chi


def refine(v, n):
    """microstructures.py:118-130 (piecewise-constant prolongation)."""
    f = n // v.shape[0]
    return np.repeat(np.repeat(v, f, axis=0), f, axis=1)


@pytest.fixture
def solid():
    return isotropic_material(2.0 / 3.0, 0.5)  # conftest.py:13-15


def test_newton_single_step_for_linear_material(solid):
    rho = G.ScalarField(G.make_grid(16), refine(laminate(8, 100.0), 16))
    rep = newton_solve(rho, np.array([1.0, 1.0, 1.0]), "green", material=solid)
    assert rep.newton_steps == 1
    assert rep.terminated == CONVERGED


def test_newton_linearity_certificate(solid):
    rho = G.ScalarField(G.make_grid(16), refine(laminate(8, 100.0), 16))
    op = make_operator(rho, solid)
    green = assemble_green(op.grid, solid)
    eb = np.array([1.0, 1.0, 1.0])
    rhs = assemble_rhs(op, eb)
    rep = pcg(op, rhs, build_preconditioner("green", op, green), green, eta=1e-10, max_iter=2000)
    recomputed = residual_force(op, rep.solution, eb)
    linear = rhs.values - apply_system(op, rep.solution).values
    assert np.abs(recomputed.values - linear).max() <= 1e-10 * np.abs(rhs.values).max()


def test_newton_zero_load_takes_zero_steps(solid):
    rho = G.ScalarField.full(G.make_grid(8), 1.0)
    rep = newton_solve(rho, np.zeros(3), "green", material=solid)
    assert rep.newton_steps == 0
    assert rep.iterations == 0


def test_newton_uniform_medium_stress(solid):
    grid = G.make_grid(8)
    rho = G.ScalarField.full(grid, 1.0)
    rep = newton_solve(rho, np.array([1.0, 1.0, 1.0]), "green", material=solid)
    op = make_operator(rho, solid)
    sig = homogenized_stress(op, rep.solution, np.array([1.0, 1.0, 1.0]))
    assert np.allclose(sig, [7.0 / 3.0, 7.0 / 3.0, 1.0], rtol=0, atol=1e-12)


@pytest.mark.parametrize("d", [2, 3])
def test_newton_solution_satisfies_tolerance(solid, d):
    eb = np.ones(3 if d == 2 else 6)
    if d == 2:
        mat = solid
        grid = G.make_grid(16)
        rho = G.ScalarField(grid, refine(cosine(8, 1e4), 16))
    else:
        mat = isotropic_material(2.0 / 3.0, 0.5, 3)
        grid = G.make_grid(16, (1.0,) * 3)
        x = np.arange(16) / 16
        v = (0.5 + 0.25 * np.cos(2 * np.pi * (x[:, None, None] - x[None, :, None]))
             * np.cos(2 * np.pi * x[None, None, :]) + 1e-4)
        rho = G.ScalarField(grid, v)
    rep = newton_solve(rho, eb, "green-jacobi", material=mat, eta=1e-6)
    assert rep.newton_steps == 1 and rep.terminated == CONVERGED
    op = make_operator(rho, mat)
    green = assemble_green(op.grid, mat)
    residual = assemble_rhs(op, eb)
    residual.values -= apply_system(op, rep.solution).values
    gnorm2 = float(np.vdot(residual.values, apply_green(green, residual).values))
    assert gnorm2 <= 1e-6 * 1.0001
    # and the device solution is the oracle's Newton solution (one PCG step)
    c = X.isotropic_stiffness(d, 2.0 / 3.0, 0.5)
    h = X.pixel_size((16,) * d, (1.0,) * d)
    blocks = X.assemble_green((16,) * d, (1.0,) * d, c)
    inv = X.assemble_jacobi(rho.values, c, h)
    f = X.residual_force(rho.values, c, h, np.zeros((d,) + (16,) * d), eb)
    it, _, term, xo = X.pcg(rho.values, c, h, f, "green-jacobi", blocks, inv)
    assert term == X.CONVERGED and abs(it - rep.iterations) <= 1
    assert np.abs(rep.solution.values - xo).max() <= 1e-8 * np.abs(xo).max()
