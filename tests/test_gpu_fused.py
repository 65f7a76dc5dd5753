"""The fused spectral passes (fused.cu) stage by stage against NumPy, and the
full fused Green / Green-Jacobi application and PCG against the oracle on
power-of-two grids (where the fused path replaces cuFFT)."""

import numpy as np
import pytest

from oracle import jfft_oracle as X
from paper_2508_02613_b200 import _native as N
from paper_2508_02613_b200 import grid as G
from paper_2508_02613_b200.material import isotropic_material
from paper_2508_02613_b200.operators import assemble_rhs, make_operator
from paper_2508_02613_b200.preconditioners import (apply_green, apply_green_jacobi,
                                                   assemble_green, assemble_jacobi,
                                                   build_preconditioner)
from paper_2508_02613_b200.solver import pcg

pytestmark = pytest.mark.gpu

SIZES = [(2, 16), (2, 32), (2, 64), (3, 16), (3, 32), (3, 64)]


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / np.abs(np.asarray(b)).max()


def full_green(bl, n, d):
    """Green blocks on the full spectrum from the rfftn-layout blocks."""
    shape = (n,) * d
    Gf = np.zeros(shape + (d, d), complex)
    for idx in np.ndindex(*shape):
        if idx[-1] <= n // 2:
            Gf[idx] = bl[idx]
        else:
            Gf[idx] = np.conj(bl[tuple((-i) % n for i in idx)])
    return Gf


@pytest.mark.parametrize("d,n", SIZES)
def test_fused_stages(d, n):
    rng = np.random.default_rng(d * 100 + n)
    grid = G.make_grid(n, (1.0,) * d)
    mat = isotropic_material(2.0 / 3.0, 0.5, d)
    green = assemble_green(grid, mat)
    u = np.ascontiguousarray(rng.normal(size=(d,) + (n,) * d))
    sh = (d, n // 2 + 1) + (n,) * (d - 1)
    call = N.load().jfftb_debug_fused_apply
    # pass A: real-to-complex along axis 0
    s1 = np.zeros(sh, complex)
    N.check(call(green.handle.ptr, None, 1, N.vptr(u), N.vptr(s1)))
    r1 = np.fft.rfft(u, axis=1)
    assert rel(s1, r1) <= 1e-14
    x = r1
    if d == 3:  # pass B: complex FFT along axis 1
        s2 = np.zeros(sh, complex)
        N.check(call(green.handle.ptr, None, 2, N.vptr(u), N.vptr(s2)))
        x = np.fft.fft(r1, axis=2)
        assert rel(s2, x) <= 1e-14
    # pass C: last-axis FFT, block solve with 1/N, last-axis inverse
    c = X.isotropic_stiffness(d, 2.0 / 3.0, 0.5)
    Gf = full_green(X.assemble_green((n,) * d, (1.0,) * d, c), n, d)[: n // 2 + 1]
    X3 = np.fft.fft(x, axis=-1)
    if d == 2:
        Z = np.einsum("xyab,bxy->axy", Gf, X3) / n ** d
    else:
        Z = np.einsum("xyzab,bxyz->axyz", Gf, X3) / n ** d
    r3 = np.fft.ifft(Z, axis=-1) * n
    s3 = np.zeros(sh, complex)
    N.check(call(green.handle.ptr, None, 3, N.vptr(u), N.vptr(s3)))
    assert rel(s3, r3) <= 1e-12
    # passes B' and I: back to real space == the oracle's apply_green
    out = np.zeros_like(u)
    N.check(call(green.handle.ptr, None, 5, N.vptr(u), N.vptr(out)))
    ref = X.apply_green(X.assemble_green((n,) * d, (1.0,) * d, c), u)
    assert rel(out, ref) <= 1e-12


@pytest.mark.parametrize("d,n", SIZES)
def test_fused_apply_and_pcg(d, n):
    rng = np.random.default_rng(7 + n + d)
    grid = G.make_grid(n, (1.0,) * d)
    mat = isotropic_material(2.0 / 3.0, 0.5, d)
    rho = rng.uniform(0.05, 2.0, (n,) * d)
    op = make_operator(G.ScalarField(grid, rho), mat)
    green = assemble_green(grid, mat)
    c = X.isotropic_stiffness(d, 2.0 / 3.0, 0.5)
    h = X.pixel_size((n,) * d, (1.0,) * d)
    bl = X.assemble_green((n,) * d, (1.0,) * d, c)
    assert np.abs(green.blocks - bl).max() <= 1e-13 * np.abs(bl).max()
    u = rng.normal(size=(d,) + (n,) * d)
    assert rel(apply_green(green, G.VectorField(grid, u)).values, X.apply_green(bl, u)) <= 1e-12
    jac = assemble_jacobi(op)
    inv = X.assemble_jacobi(rho, c, h)
    gj = apply_green_jacobi(jac, green, G.VectorField(grid, u)).values
    assert rel(gj, inv * X.apply_green(bl, inv * u)) <= 1e-12
    eb = np.ones(3 if d == 2 else 6)
    rhs = assemble_rhs(op, eb)
    f = X.assemble_rhs(rho, c, h, eb)
    for kind in X.KINDS:
        rep = pcg(op, rhs, build_preconditioner(kind, op, green), green, eta=1e-10)
        it, hist, term, x = X.pcg(rho, c, h, f, kind, bl, inv, eta=1e-10)
        assert abs(rep.iterations - it) <= 1, kind
        # field parity: 1e-9, or 10x the CPU-vs-CPU round-off floor of this
        # solve (the oracle against itself with exactly rounded dots) when
        # the recurrence amplifies round-off beyond that
        floor = floor_dev(rho, c, h, f, kind, bl, inv, x)
        assert rel(rep.solution.values, x) <= max(1e-9, 10 * floor), (kind, floor)
        assert rel(rep.residual_history[:3], hist[:3]) <= 1e-10, kind


def floor_dev(rho, c, h, f, kind, bl, inv, x):
    import math
    orig = X._dot
    X._dot = lambda a, b: math.fsum((a * b).ravel())
    try:
        _, _, _, x2 = X.pcg(rho, c, h, f, kind, bl, inv, eta=1e-10)
    finally:
        X._dot = orig
    return rel(x2, x)


def test_analytic_green_blocks_match_stored():
    """The closed-form 3-D Green blocks (JFFTB_GREEN_ANALYTIC=1, fused.cu
    green_block) against the stored pseudo-inverse through a full fused
    application, in a fresh process (the switch is read once)."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, sys
sys.path.insert(0, sys.argv[1])
from oracle import jfft_oracle as X
from paper_2508_02613_b200 import grid as G
from paper_2508_02613_b200.material import isotropic_material
from paper_2508_02613_b200.preconditioners import apply_green, assemble_green
n, lengths = 32, (1.0, 2.0, 0.5)
grid = G.make_grid(n, lengths)
mat = isotropic_material(0.7, 0.4, 3)
green = assemble_green(grid, mat)
u = np.random.default_rng(4).normal(size=(3, n, n, n))
out = apply_green(green, G.VectorField(grid, u)).values
ref = X.apply_green(X.assemble_green((n,) * 3, lengths, X.isotropic_stiffness(3, 0.7, 0.4)), u)
err = np.abs(out - ref).max() / np.abs(ref).max()
assert err <= 1e-12, err
print("ok", err)
'''
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, JFFTB_GREEN_ANALYTIC="1")
    r = subprocess.run([sys.executable, "-c", code, repo], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("n,kind", [(32, "green-jacobi"), (64, "green-jacobi"), (64, "green"),
                                    (128, "green-jacobi")])
def test_merged_spectral_kernel_matches_separate_passes(n, kind, monkeypatch):
    """JFFTB_BCB=1 runs passes B, C and B' as one persistent kernel that chains
    the k0 planes through L2 (fused.cu passBCB).  Same transforms and block
    solve, other Parseval grouping: histories to 1e-12, fields to 1e-11, and
    bitwise equal to itself on a rerun (the item -> CTA map is dynamic, the
    sums are not)."""
    from paper_2508_02613_b200 import microstructures as ms
    lam, mu = ms.lame_from_poisson()
    rho = ms.random_spheres(n, count=5, rmin=n / 10, rmax=n / 5, filters=3, emin=1e-2, seed=n)
    grid = G.make_grid(n, (1.0,) * 3)
    mat = isotropic_material(lam, mu, 3)
    eb = np.array([0.4, -0.1, 0.2, 0.3, 0.0, 0.5])
    reps = []
    for flag in ("0", "1", "1"):
        monkeypatch.setenv("JFFTB_BCB", flag)
        op = make_operator(G.ScalarField(grid, rho), mat)
        green = assemble_green(grid, mat)
        rhs = assemble_rhs(op, eb)
        reps.append(pcg(op, rhs, build_preconditioner(kind, op, green), green, eta=0.0,
                        max_iter=15))
    base, merged, again = reps
    assert merged.iterations == base.iterations == 15
    assert rel(merged.residual_history, base.residual_history) <= 1e-12
    assert rel(merged.solution.values, base.solution.values) <= 1e-11
    assert merged.residual_history == again.residual_history
    assert np.array_equal(merged.solution.values, again.solution.values)
