"""Load-case solves for homogenisation / topology optimisation on the device
(the reference's topopt.py:98-196 consumer of ``pcg``).

``solve_load_cases`` equilibrates a set of macroscopic loads (by default the
Mandel basis, as ``topopt._solve_load_cases`` does) against one operator,
one preconditioner and one Green operator: every right-hand side is
assembled, solved and paired in device memory, and only the load-by-load
stress matrix (and, on request, the solutions) come back to the host.  The
stress matrix is the reference's energy form ``_stress_matrix``
(topopt.py:136-141) -- quadratically accurate in the solver error --
and ``pairing_field`` is the per-voxel contraction of the pairings with a
load-pair weight matrix that ``_stress_gradient`` (topopt.py:163-180) needs.

The reference stops a load case at the iteration cap only when its final
squared Green norm exceeds 1e3 * eta (topopt.py:120-125); so does this.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .grid import mandel_dim
from .operators import grid_dim, op_handle
from .solver import (CONVERGED, DEFAULT_ETA_CG, DEFAULT_MAX_ITER, SolverAbortError, pcg_device,
                     pcg_device_batch)


@dataclass
class LoadCaseReport:
    stress: np.ndarray                 # (L, L) energy-form homogenised stress
    iterations: list                   # PCG iterations per load case
    terminated: list                   # "converged" / "iteration-cap" per case
    residual_history: list             # per case, iterations + 1 entries
    loads: np.ndarray                  # (L, M) macroscopic strains (Mandel)
    solutions: object = field(default=None, repr=False)  # (L, d, n...) tensor on the device


def _torch():
    import torch
    return torch


def solve_load_cases(op, preconditioner, green, loads=None, eta: float = DEFAULT_ETA_CG,
                     max_iter: int = DEFAULT_MAX_ITER, keep_solutions: bool = False,
                     cap_tolerance: float = 1e3, batch: bool = True) -> LoadCaseReport:
    """Solve K u_g = f(Ebar_g) for every load g (topopt.py:98-127).

    ``loads``: (L, M) Mandel strains, L <= 6 (default: the M unit loads).
    ``batch``: run the L solves side by side (jfftb_pcg_batch) where the
    grid and kind allow it; each solve keeps its own termination.
    Returns a :class:`LoadCaseReport`; with ``keep_solutions`` its
    ``solutions`` is the (L, d, n, ...) float64 CUDA tensor of the solves.
    """
    torch = _torch()
    d = grid_dim(op.grid)
    M = mandel_dim(d)
    E = np.eye(M) if loads is None else np.array(loads, dtype=np.float64, ndmin=2)
    if E.ndim != 2 or E.shape[1] != M or not 1 <= E.shape[0] <= 6:
        raise ValueError(f"loads must be (L, {M}) with 1 <= L <= 6, got {E.shape}")
    if not np.all(np.isfinite(E)):
        raise ValueError("macroscopic strain must be finite")
    L = E.shape[0]
    h = op_handle(op)
    lib = N.load()
    dev = torch.device("cuda", N.device_id())
    shape = (d,) + (op.grid.n,) * d
    us = torch.empty((L,) + shape, dtype=torch.float64, device=dev)
    kind = preconditioner.kind
    from .preconditioners import green_handle, jacobi_handle
    green_pc = green_handle(preconditioner.green) if preconditioner.green is not None else None
    jac = jacobi_handle(preconditioner.jacobi) if preconditioner.jacobi is not None else None
    green_h = green_handle(green)
    n = op.grid.n
    # batched: every stage of the L solves in one launch (3-D power-of-two
    # grids, spectral kinds); otherwise one solve after the other
    batched = (batch and d == 3 and kind in ("green", "green-jacobi") and 16 <= n <= 2048
               and n & (n - 1) == 0)
    rhs = torch.empty(((L,) if batched else ()) + shape, dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    results = []
    for g in range(L):
        e = np.ascontiguousarray(E[g])
        dst = rhs[g] if batched else rhs
        N.check(lib.jfftb_assemble_rhs(h.ptr, N.dptr(e), C.c_void_p(dst.data_ptr()), N.DEVICE))
        if not batched:
            it, hist, term, _ = pcg_device(h, kind, green_h, jac, rhs.data_ptr(),
                                           us[g].data_ptr(), eta, max_iter, green_pc_h=green_pc)
            results.append((it, hist, term))
    if batched:
        results, _ = pcg_device_batch(h, kind, green_h, jac, L, rhs.data_ptr(),
                                      us.data_ptr(), eta, max_iter, green_pc_h=green_pc)
    its, terms, hists = [], [], []
    for g, (it, hist, term) in enumerate(results):
        if term != CONVERGED and hist[-1] > cap_tolerance * eta:
            raise SolverAbortError(
                f"load case {g}: iteration cap {max_iter} reached with squared Green norm "
                f"{hist[-1]:.3e}")
        its.append(it)
        terms.append(term)
        hists.append(hist)
    sigma = np.zeros((L, L))
    N.check(lib.jfftb_load_pairings(h.ptr, L, C.c_void_p(us.data_ptr()), N.dptr(E), None,
                                    N.dptr(sigma), None, N.DEVICE))
    return LoadCaseReport(sigma, its, terms, hists, E, us if keep_solutions else None)


def pairing_field(op, solutions, loads, weights):
    """sum_gc weights[g, c] * sum_t eps_c^T C0 eps_g per voxel (topopt.py:
    130-133 and 163-180 before the scale): ``solutions`` is the device
    tensor of :func:`solve_load_cases`; returns a host array of the grid's
    shape."""
    torch = _torch()
    d = grid_dim(op.grid)
    E = np.ascontiguousarray(np.array(loads, dtype=np.float64, ndmin=2))
    W = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    L = E.shape[0]
    if W.shape != (L, L):
        raise ValueError(f"weights must be ({L}, {L})")
    if tuple(solutions.shape) != (L, d) + (op.grid.n,) * d:
        raise ValueError("solutions do not match the loads and the grid")
    out = torch.empty((op.grid.n,) * d, dtype=torch.float64, device=solutions.device)
    sigma = np.zeros((L, L))
    torch.cuda.synchronize(solutions.device)
    N.check(N.load().jfftb_load_pairings(op_handle(op).ptr, L,
                                         C.c_void_p(solutions.contiguous().data_ptr()),
                                         N.dptr(E), N.dptr(W), N.dptr(sigma),
                                         C.c_void_p(out.data_ptr()), N.DEVICE))
    return out.cpu().numpy()


def _bench(n: int = 128, kind: str = "green-jacobi"):  # pragma: no cover
    # python -m paper_2508_02613_b200.loadcases [n] [kind]
    """Six 3-D load cases on BASELINE config 3 (128^3 spheres): wall time of
    the device driver (assembly, solves, pairings) and its throughput."""
    import json
    import time

    from . import grid as G
    from . import microstructures as ms
    from .material import isotropic_material
    from .operators import make_operator
    from .preconditioners import assemble_green, build_preconditioner
    lam, mu = ms.lame_from_poisson()
    rho = ms.random_spheres(n, seed=0)
    grid = G.make_grid(n, (1.0,) * 3)
    mat = isotropic_material(lam, mu, 3)
    op = make_operator(G.ScalarField(grid, rho), mat)
    green = assemble_green(grid, mat)
    pc = build_preconditioner(kind, op, green)
    out = {"what": f"6 load cases, config 3 ({n}^3 spheres), {kind}, eta 1e-6"}
    for batch in (True, False, True, False):
        solve_load_cases(op, pc, green, loads=np.eye(6)[:2], max_iter=5, cap_tolerance=1e300,
                         batch=batch)
        _torch().cuda.synchronize()
        t0 = time.perf_counter()
        rep = solve_load_cases(op, pc, green, batch=batch)
        dt = time.perf_counter() - t0
        its = sum(rep.iterations)
        out["batched" if batch else "sequential"] = {
            "seconds": dt, "iterations": rep.iterations,
            "GDOF_it_per_s": 3 * n ** 3 * its / dt / 1e9,
            "stress_diag": np.diag(rep.stress).tolist()}
    print(json.dumps(out))


if __name__ == "__main__":  # pragma: no cover
    import sys
    _bench(*([int(sys.argv[1])] if len(sys.argv) > 1 else []) +
           ([sys.argv[2]] if len(sys.argv) > 2 else []))
