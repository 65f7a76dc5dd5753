"""Small case for compute-sanitizer (racecheck / synccheck): 64^3 Green-Jacobi
PCG (stencil, passes A3/B/C/B'/I, reductions), K u, and a loopback P = 2
distributed solve, on cuda:0.  Run as
    compute-sanitizer --tool racecheck python profiles/sanitize_case.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(
    os.path.abspath(__file__)))))
os.environ.setdefault("JFFTB_GRAPHS", "0")
from paper_2508_02613_b200 import dist as Dm  # noqa: E402
from paper_2508_02613_b200 import grid as G  # noqa: E402
from paper_2508_02613_b200 import microstructures as ms  # noqa: E402
from paper_2508_02613_b200.material import isotropic_material  # noqa: E402
from paper_2508_02613_b200.operators import apply_system, assemble_rhs, make_operator  # noqa: E402
from paper_2508_02613_b200.preconditioners import assemble_green, build_preconditioner  # noqa: E402
from paper_2508_02613_b200.solver import pcg  # noqa: E402

n = 64
lam, mu = ms.lame_from_poisson()
rho = ms.random_spheres(n, count=6, rmin=4, rmax=10, filters=2, emin=1e-2, seed=1)
grid = G.make_grid(n, (1.0,) * 3)
mat = isotropic_material(lam, mu, 3)
op = make_operator(G.ScalarField(grid, rho), mat)
green = assemble_green(grid, mat)
rhs = assemble_rhs(op, np.array([1.0, 0, 0, 0, 0, 0]))
for kind in ("green-jacobi", "green"):
    rep = pcg(op, rhs, build_preconditioner(kind, op, green), green, eta=0.0, max_iter=3)
    print(kind, rep.iterations, rep.residual_history[-1])
ku = apply_system(op, rep.solution)
comm = Dm.Comm.local_ranks(2)
D = Dm.DistSolver(comm, (n,) * 3, (1.0,) * 3, np.stack(Dm.split(rho, 2, axis=1)), lam, mu)
rep = D.pcg(D.assemble_rhs(np.array([1.0, 0, 0, 0, 0, 0])), eta=0.0, max_iter=3)
print("dist", rep.iterations, rep.residual_history[-1])
