"""Device load-case driver (loadcases.py, csrc/loadcases.cu) against the
oracle's restatement of topopt.py:98-180 (pinned to the reference in
test_oracle_pins.py::test_load_case_pairings_match_reference)."""

import numpy as np
import pytest

from oracle import jfft_oracle as X
from paper_2508_02613_b200 import grid as G
from paper_2508_02613_b200 import microstructures as ms
from paper_2508_02613_b200.loadcases import pairing_field, solve_load_cases
from paper_2508_02613_b200.material import isotropic_material
from paper_2508_02613_b200.operators import make_operator
from paper_2508_02613_b200.preconditioners import assemble_green, build_preconditioner
from paper_2508_02613_b200.solver import SolverAbortError

pytestmark = pytest.mark.gpu


def _problem(d, n, seed):
    lam, mu = ms.lame_from_poisson()
    if d == 2:
        rho = ms.bernoulli_smoothed(n, 10, 1e3, seed)
    else:
        rho = ms.random_spheres(n, count=4, rmin=2.0, rmax=5.0, filters=3, seed=seed)
    lengths = (1.0,) * d
    grid = G.make_grid(n, lengths)
    mat = isotropic_material(lam, mu, d)
    op = make_operator(G.ScalarField(grid, rho), mat)
    return rho, lam, mu, lengths, grid, mat, op


@pytest.mark.parametrize("d,n,kind", [(2, 32, "green"), (2, 48, "green-jacobi"),
                                      (3, 16, "green-jacobi"), (3, 16, "green")])
def test_stress_matrix_and_counts(d, n, kind):
    rho, lam, mu, lengths, grid, mat, op = _problem(d, n, 1)
    green = assemble_green(grid, mat)
    rep = solve_load_cases(op, build_preconditioner(kind, op, green), green,
                           keep_solutions=True)
    c = X.isotropic_stiffness(d, lam, mu)
    h = X.pixel_size((n,) * d, lengths)
    blocks = X.assemble_green((n,) * d, lengths, c)
    inv = X.assemble_jacobi(rho, c, h) if kind == "green-jacobi" else None
    M = c.shape[0]
    us = []
    for g, e in enumerate(np.eye(M)):
        f = X.assemble_rhs(rho, c, h, e)
        it, hist, term, x = X.pcg(rho, c, h, f, kind, blocks, inv)
        assert abs(rep.iterations[g] - it) <= 1, (g, rep.iterations[g], it)
        us.append(x)
    sig_ref = X.stress_matrix(rho, c, h, us, np.eye(M), lengths)
    assert np.abs(rep.stress - sig_ref).max() <= 1e-9 * np.abs(sig_ref).max()
    assert np.allclose(rep.stress, rep.stress.T, rtol=0, atol=0)
    # the solutions themselves (zero mean, as pcg returns them)
    got = rep.solutions.cpu().numpy()
    for g in range(M):
        assert np.abs(got[g] - us[g]).max() <= 1e-8 * np.abs(us[g]).max()
    # uniform density = C0 in the energy form (known answer)
    W = np.random.default_rng(0).normal(size=(M, M))
    fld = pairing_field(op, rep.solutions, np.eye(M), W)
    P = X.strain_pairings(c, h, us, np.eye(M))
    ref = np.einsum("gc,gc...->...", W, P)
    assert np.abs(fld - ref).max() <= 1e-9 * np.abs(ref).max()


def test_uniform_medium_gives_c0():
    d, n = 3, 8
    grid = G.make_grid(n, (1.0, 2.0, 0.5))
    lam, mu = 0.7, 0.4
    mat = isotropic_material(lam, mu, d)
    op = make_operator(G.ScalarField(grid, np.full((n,) * d, 2.5)), mat)
    green = assemble_green(grid, mat)
    rep = solve_load_cases(op, build_preconditioner("green", op, green), green)
    assert np.allclose(rep.stress, 2.5 * X.isotropic_stiffness(d, lam, mu), rtol=1e-12,
                       atol=1e-12)
    assert rep.iterations == [0] * 6 or max(rep.iterations) <= 1


def test_cap_policy_and_validation():
    rho, lam, mu, lengths, grid, mat, op = _problem(2, 32, 2)
    green = assemble_green(grid, mat)
    pc = build_preconditioner("none", op, green)
    with pytest.raises(SolverAbortError):
        solve_load_cases(op, pc, green, max_iter=2)
    # a loose cap tolerance lets capped cases through (topopt.py:120-125)
    rep = solve_load_cases(op, pc, green, max_iter=2, cap_tolerance=1e300)
    assert rep.terminated == ["iteration-cap"] * 3
    with pytest.raises(ValueError):
        solve_load_cases(op, pc, green, loads=np.ones((7, 3)))
    with pytest.raises(ValueError):
        solve_load_cases(op, pc, green, loads=np.ones((2, 6)))


@pytest.mark.parametrize("kind", ["green-jacobi", "green"])
def test_batched_matches_sequential(kind):
    """jfftb_pcg_batch (one launch per stage for all load cases) against the
    same solves one after the other: same iteration counts, histories and
    solutions to round-off (the batched pass C reduces over a different
    number of blocks), same stress matrix."""
    rho, lam, mu, lengths, grid, mat, op = _problem(3, 32, 3)
    green = assemble_green(grid, mat)
    pc = build_preconditioner(kind, op, green)
    loads = np.eye(6)[[0, 2, 5]]
    a = solve_load_cases(op, pc, green, loads=loads, keep_solutions=True, batch=True)
    b = solve_load_cases(op, pc, green, loads=loads, keep_solutions=True, batch=False)
    for g in range(3):
        assert abs(a.iterations[g] - b.iterations[g]) <= 1
        k = min(len(a.residual_history[g]), len(b.residual_history[g]), 10)
        ha, hb = np.array(a.residual_history[g][:k]), np.array(b.residual_history[g][:k])
        assert np.abs(ha - hb).max() <= 1e-12 * hb[0]
    assert np.abs(a.stress - b.stress).max() <= 1e-9 * np.abs(b.stress).max()
    ua, ub = a.solutions.cpu().numpy(), b.solutions.cpu().numpy()
    assert np.abs(ua - ub).max() <= 1e-7 * np.abs(ub).max()
