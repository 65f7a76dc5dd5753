"""Generate the golden fixtures under tests/golden/.

2-D fixtures come from the REFERENCE itself (the ``jfft`` package, imported
from /root/reference/pkg/src in the build container -- it does not travel to
the GPU box, so its outputs are committed here).  3-D fixtures come from the
oracle restatement (oracle/jfft_oracle.py), which the 2-D fixtures pin.

Usage:  python tests/golden/make_golden.py [small|config1|config2|config3|all]

config2 (2048^2, eight reference solves incl. a 999-iteration capped run)
takes ~30 min of CPU; the others finish in about a minute.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from oracle import jfft_oracle as X  # noqa: E402
from paper_2508_02613_b200 import microstructures as ms  # noqa: E402


def _ref():
    import jfft  # noqa: F401
    from jfft import grid, material, microstructures, operators, preconditioners, solver
    return grid, material, microstructures, operators, preconditioners, solver


def ref_input_2d(n, filters, chi, seed):
    """The config-1/2 density built with the reference's own filter and
    rescale; asserts our generator reproduces it bit for bit."""
    G, _, M, _, _, _ = _ref()
    rng = np.random.default_rng(seed)
    v = (rng.random((n, n)) < 0.5).astype(float)
    f = G.ScalarField(G.make_grid(n), v)
    for _ in range(filters):
        f = M.gaussian_filter(f)
    f = M.rescale_contrast(f, chi)
    ours = ms.bernoulli_smoothed(n, filters, chi, seed)
    assert np.array_equal(ours, f.values), "generator drifted from the reference"
    return f.values


def ref_solve(rho, eps_bar, kind, lam, mu, eta=1e-6, cap=999, green=None):
    G, Mat, _, O, P, S = _ref()
    n = rho.shape[0]
    grid = G.make_grid(n)
    mat = Mat.isotropic_material(lam, mu)
    op = O.make_operator(G.ScalarField(grid, rho), mat)
    if green is None:
        green = P.assemble_green(grid, mat)
    pre = P.build_preconditioner(kind, op, green)
    rhs = O.assemble_rhs(op, eps_bar)
    t0 = time.perf_counter()
    rep = S.pcg(op, rhs, pre, green, eta=eta, max_iter=cap)
    wall = time.perf_counter() - t0
    sig = O.homogenized_stress(op, rep.solution, eps_bar)
    return rep, sig, wall, green


def make_small():
    G, Mat, _, O, P, S = _ref()
    out = {}
    mat = Mat.isotropic_material(2.0 / 3.0, 0.5)
    for n, lengths, seed in ((8, (1.0, 2.0), 1), (16, (1.0, 1.0), 2), (6, (2.0, 0.5), 3)):
        rng = np.random.default_rng(seed)
        grid = G.make_grid(n, lengths)
        rho = rng.uniform(0.05, 2.0, (n, n))
        op = O.make_operator(G.ScalarField(grid, rho), mat)
        u = rng.normal(size=(2, n, n))
        eb = np.array([1.0, -0.5, 0.3])
        key = f"n{n}"
        out[f"{key}_lengths"] = np.array(lengths)
        out[f"{key}_rho"] = rho
        out[f"{key}_u"] = u
        out[f"{key}_Ku"] = O.apply_system(op, G.VectorField(grid, u)).values
        out[f"{key}_eps_bar"] = eb
        out[f"{key}_rhs"] = O.assemble_rhs(op, eb).values
        out[f"{key}_strain"] = O.total_strain(op, G.VectorField(grid, u), eb).values
        out[f"{key}_sigma"] = O.homogenized_stress(op, G.VectorField(grid, u), eb)
        out[f"{key}_resforce"] = O.residual_force(op, G.VectorField(grid, u), eb).values
        green = P.assemble_green(grid, mat)
        out[f"{key}_blocks"] = green.blocks
        out[f"{key}_Gu"] = P.apply_green(green, G.VectorField(grid, u)).values
        if n % 2 == 0:
            jac = P.assemble_jacobi(op)
            out[f"{key}_inv_sqrt"] = jac.inv_sqrt
            out[f"{key}_GJu"] = P.apply_green_jacobi(jac, green, G.VectorField(grid, u)).values
            rhs = O.assemble_rhs(op, eb)
            for kind in ("none", "green", "jacobi", "green-jacobi"):
                rep = S.pcg(op, rhs, P.build_preconditioner(kind, op, green), green,
                            eta=1e-10, max_iter=999)
                out[f"{key}_{kind}_iters"] = np.array(rep.iterations)
                out[f"{key}_{kind}_hist"] = np.array(rep.residual_history)
                out[f"{key}_{kind}_x"] = rep.solution.values
    np.savez_compressed(os.path.join(HERE, "small2d.npz"), **out)
    print("small2d.npz", len(out), "arrays")

    # 3-D: oracle restatement (no reference implementation exists in 3-D)
    out = {}
    for n, lengths, seed in (((4, 4, 4), (1.0, 1.5, 0.75), 4), ((6, 4, 8), (1.0, 1.0, 2.0), 5)):
        rng = np.random.default_rng(seed)
        c = X.isotropic_stiffness(3, 2.0 / 3.0, 0.5)
        h = X.pixel_size(n, lengths)
        rho = rng.uniform(0.05, 2.0, n)
        u = rng.normal(size=(3,) + n)
        eb = np.array([1.0, -0.5, 0.3, 0.2, -0.1, 0.4])
        key = "n" + "x".join(map(str, n))
        out[f"{key}_lengths"] = np.array(lengths)
        out[f"{key}_rho"] = rho
        out[f"{key}_u"] = u
        out[f"{key}_Ku"] = X.apply_K(rho, c, h, u)
        out[f"{key}_eps_bar"] = eb
        out[f"{key}_rhs"] = X.assemble_rhs(rho, c, h, eb)
        out[f"{key}_strain"] = X.total_strain(h, u, eb)
        out[f"{key}_sigma"] = X.homogenized_stress(rho, c, h, u, eb, lengths)
        blocks = X.assemble_green(n, lengths, c)
        out[f"{key}_blocks"] = blocks
        out[f"{key}_Gu"] = X.apply_green(blocks, u)
        inv_sqrt = X.assemble_jacobi(rho, c, h)
        out[f"{key}_inv_sqrt"] = inv_sqrt
        rhs = X.assemble_rhs(rho, c, h, eb)
        for kind in X.KINDS:
            it, hist, term, x = X.pcg(rho, c, h, rhs, kind, blocks, inv_sqrt, eta=1e-10)
            out[f"{key}_{kind}_iters"] = np.array(it)
            out[f"{key}_{kind}_hist"] = np.array(hist)
            out[f"{key}_{kind}_x"] = x
    np.savez_compressed(os.path.join(HERE, "small3d.npz"), **out)
    print("small3d.npz", len(out), "arrays")


def make_config1():
    lam, mu = ms.lame_from_poisson()
    out = {"lam": lam, "mu": mu}
    eb = np.array([1.0, 0.0, 0.0])
    green = None
    for filters in (10, 0):
        rho = ref_input_2d(256, filters, 1e4, 0)
        for kind in ("green", "green-jacobi"):
            rep, sig, wall, green = ref_solve(rho, eb, kind, lam, mu, green=green)
            key = f"i{filters}_{kind}"
            out[f"{key}_iters"] = rep.iterations
            out[f"{key}_hist"] = rep.residual_history
            out[f"{key}_terminated"] = rep.terminated
            out[f"{key}_sigma"] = sig.tolist()
            out[f"{key}_wall"] = wall
            out[f"{key}_unorm"] = float(np.linalg.norm(rep.solution.values))
            if filters == 10:
                np.save(os.path.join(HERE, f"config1_{key}_u.npy"),
                        rep.solution.values.astype("<f8"))
            if rep.terminated != "converged":
                # CPU-vs-CPU round-off floor of a capped run: the reference
                # itself with exactly rounded dot products (math.fsum)
                import math
                from jfft import solver as S
                orig = S._dot
                S._dot = lambda a, b: math.fsum((a.values * b.values).ravel())
                try:
                    rep2, sig2, _, _ = ref_solve(rho, eb, kind, lam, mu, green=green)
                finally:
                    S._dot = orig
                out[f"{key}_fsum_hist"] = rep2.residual_history
                out[f"{key}_fsum_sigma"] = sig2.tolist()
                out[f"{key}_fsum_iters"] = rep2.iterations
            print(key, rep.iterations, rep.terminated, sig, f"{wall:.1f}s", flush=True)
    with open(os.path.join(HERE, "config1.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def make_config2():
    lam, mu = ms.lame_from_poisson()
    eb = ms.mandel_shear(2, 0, 1, 0.5)
    path = os.path.join(HERE, "config2.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    out.update({"lam": lam, "mu": mu, "eps_bar": eb.tolist(), "n": 2048})
    green = None
    for filters in (50, 20, 5, 0):
        rho = ref_input_2d(2048, filters, 1e4, 0)
        for kind in ("green", "green-jacobi"):
            key = f"i{filters}_{kind}"
            if f"{key}_iters" in out:
                continue
            rep, sig, wall, green = ref_solve(rho, eb, kind, lam, mu, green=green)
            u = rep.solution.values
            out[f"{key}_iters"] = rep.iterations
            out[f"{key}_hist"] = rep.residual_history
            out[f"{key}_terminated"] = rep.terminated
            out[f"{key}_sigma"] = sig.tolist()
            out[f"{key}_wall"] = wall
            out[f"{key}_unorm"] = float(np.linalg.norm(u))
            out[f"{key}_usample"] = u[:, ::256, ::256].tolist()
            print(key, rep.iterations, rep.terminated, sig, f"{wall:.1f}s", flush=True)
            with open(path, "w") as fh:
                json.dump(out, fh, indent=1)


def make_config3():
    """3-D 128^3 spheres (BASELINE config 3) through the oracle."""
    lam, mu = ms.lame_from_poisson()
    n = (128, 128, 128)
    rho = ms.random_spheres(128, seed=0)
    c = X.isotropic_stiffness(3, lam, mu)
    h = X.pixel_size(n, (1.0, 1.0, 1.0))
    eb = np.array([1.0, 0, 0, 0, 0, 0])
    blocks = X.assemble_green(n, (1.0, 1.0, 1.0), c)
    inv_sqrt = X.assemble_jacobi(rho, c, h)
    rhs = X.assemble_rhs(rho, c, h, eb)
    out = {"lam": lam, "mu": mu, "rho_sum": float(rho.sum()), "rho_min": float(rho.min()),
           "rho_max": float(rho.max())}
    for kind in ("green", "green-jacobi"):
        t0 = time.perf_counter()
        it, hist, term, x = X.pcg(rho, c, h, rhs, kind, blocks, inv_sqrt)
        wall = time.perf_counter() - t0
        sig = X.homogenized_stress(rho, c, h, x, eb, (1.0, 1.0, 1.0))
        key = kind
        out[f"{key}_iters"] = it
        out[f"{key}_hist"] = hist
        out[f"{key}_terminated"] = term
        out[f"{key}_sigma"] = sig.tolist()
        out[f"{key}_wall"] = wall
        out[f"{key}_unorm"] = float(np.linalg.norm(x))
        out[f"{key}_usample"] = x[:, ::16, ::16, ::16].tolist()
        print(kind, it, term, sig, f"{wall:.1f}s", flush=True)
    with open(os.path.join(HERE, "config3.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def _fsum_dot():
    import math
    return lambda a, b: math.fsum((np.asarray(a) * np.asarray(b)).ravel())


def make_floors():
    """CPU-vs-CPU round-off floor of the long Green-Jacobi solves: the same
    solver with exactly rounded dot products (math.fsum).  A GPU result is
    held to max(1e-9, 10 x floor) -- two correct implementations with
    different summation orders differ by about the floor, which Green-Jacobi
    amplifies to ~1e-6 .. 1e-3 on 50-165-iteration solves."""
    import math
    from jfft import solver as S
    lam, mu = ms.lame_from_poisson()
    # config 2 (reference, 2-D)
    path = os.path.join(HERE, "config2.json")
    out = json.load(open(path))
    eb = np.array(out["eps_bar"])
    green = None
    for filters in (50, 20, 5):
        key = f"i{filters}_green-jacobi"
        if f"{key}_fsum_unorm" in out:
            continue
        rho = ref_input_2d(2048, filters, 1e4, 0)
        orig = S._dot
        S._dot = lambda a, b: math.fsum((a.values * b.values).ravel())
        try:
            rep, sig, wall, green = ref_solve(rho, eb, "green-jacobi", lam, mu, green=green)
        finally:
            S._dot = orig
        u = rep.solution.values
        out[f"{key}_fsum_iters"] = rep.iterations
        out[f"{key}_fsum_sigma"] = sig.tolist()
        out[f"{key}_fsum_unorm"] = float(np.linalg.norm(u))
        out[f"{key}_fsum_usample"] = u[:, ::256, ::256].tolist()
        print("floor", key, rep.iterations, f"{wall:.0f}s", flush=True)
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1)
    # config 3 (oracle, 3-D)
    path = os.path.join(HERE, "config3.json")
    out = json.load(open(path))
    if "green-jacobi_fsum_unorm" not in out:
        n = (128, 128, 128)
        rho = ms.random_spheres(128, seed=0)
        c = X.isotropic_stiffness(3, lam, mu)
        h = X.pixel_size(n, (1.0, 1.0, 1.0))
        eb3 = np.array([1.0, 0, 0, 0, 0, 0])
        blocks = X.assemble_green(n, (1.0, 1.0, 1.0), c)
        inv_sqrt = X.assemble_jacobi(rho, c, h)
        rhs = X.assemble_rhs(rho, c, h, eb3)
        orig = X._dot
        X._dot = lambda a, b: math.fsum((a * b).ravel())
        try:
            it, hist, term, x = X.pcg(rho, c, h, rhs, "green-jacobi", blocks, inv_sqrt)
        finally:
            X._dot = orig
        sig = X.homogenized_stress(rho, c, h, x, eb3, (1.0, 1.0, 1.0))
        out["green-jacobi_fsum_iters"] = it
        out["green-jacobi_fsum_sigma"] = sig.tolist()
        out["green-jacobi_fsum_unorm"] = float(np.linalg.norm(x))
        out["green-jacobi_fsum_usample"] = x[:, ::16, ::16, ::16].tolist()
        print("floor config3", it, flush=True)
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what == "floors":
        make_floors()
    if what in ("small", "all"):
        make_small()
    if what in ("config1", "all"):
        make_config1()
    if what in ("config3", "all"):
        make_config3()
    if what in ("config2", "all"):
        make_config2()
