"""Pin the CPU oracle (oracle/jfft_oracle.py) before trusting it:

* d = 2 against fixtures produced by the REFERENCE itself
  (tests/golden/make_golden.py ran /root/reference/pkg/src/jfft): bit-exact;
* d = 3 (no reference exists) against first-principles known answers: a
  dense stiffness assembled from P1 shape functions of the Kuhn tetrahedra,
  symmetry, the rigid-translation null space, uniform-medium stress, the
  laminate closed form, and G K_ref = I - mean.
"""

import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle import jfft_oracle as X

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


@pytest.fixture(scope="module")
def small2d():
    return np.load(os.path.join(GOLD, "small2d.npz"))


@pytest.mark.parametrize("key", ["n8", "n16", "n6"])
def test_oracle_2d_matches_reference_bitwise(small2d, key):
    rho = small2d[f"{key}_rho"]
    n = rho.shape
    lengths = tuple(small2d[f"{key}_lengths"])
    h = X.pixel_size(n, lengths)
    c = X.isotropic_stiffness(2, 2.0 / 3.0, 0.5)
    u = small2d[f"{key}_u"]
    eb = small2d[f"{key}_eps_bar"]
    assert np.array_equal(X.apply_K(rho, c, h, u), small2d[f"{key}_Ku"])
    assert np.array_equal(X.assemble_rhs(rho, c, h, eb), small2d[f"{key}_rhs"])
    assert np.array_equal(X.total_strain(h, u, eb), small2d[f"{key}_strain"])
    assert np.array_equal(X.residual_force(rho, c, h, u, eb), small2d[f"{key}_resforce"])
    assert np.array_equal(X.homogenized_stress(rho, c, h, u, eb, lengths),
                          small2d[f"{key}_sigma"])
    blocks = X.assemble_green(n, lengths, c)
    assert np.array_equal(blocks, small2d[f"{key}_blocks"])
    assert np.array_equal(X.apply_green(blocks, u), small2d[f"{key}_Gu"])
    if n[0] % 2 == 0:
        inv = X.assemble_jacobi(rho, c, h)
        assert np.array_equal(inv, small2d[f"{key}_inv_sqrt"])
        f = X.assemble_rhs(rho, c, h, eb)
        for kind in X.KINDS:
            it, hist, term, x = X.pcg(rho, c, h, f, kind, blocks, inv, eta=1e-10)
            assert it == int(small2d[f"{key}_{kind}_iters"])
            assert np.array_equal(np.array(hist), small2d[f"{key}_{kind}_hist"])
            assert np.array_equal(x, small2d[f"{key}_{kind}_x"])


def test_oracle_config1_matches_reference():
    """BASELINE config 1 (256^2) iteration counts, histories, stress and field."""
    from paper_2508_02613_b200 import microstructures as ms
    gold = json.load(open(os.path.join(GOLD, "config1.json")))
    lam, mu = gold["lam"], gold["mu"]
    rho = ms.bernoulli_smoothed(256, 10, 1e4, 0)
    c = X.isotropic_stiffness(2, lam, mu)
    h = X.pixel_size((256, 256), (1.0, 1.0))
    blocks = X.assemble_green((256, 256), (1.0, 1.0), c)
    inv = X.assemble_jacobi(rho, c, h)
    eb = np.array([1.0, 0.0, 0.0])
    f = X.assemble_rhs(rho, c, h, eb)
    for kind in ("green", "green-jacobi"):
        key = f"i10_{kind}"
        it, hist, term, x = X.pcg(rho, c, h, f, kind, blocks, inv)
        assert it == gold[f"{key}_iters"]
        assert term == gold[f"{key}_terminated"]
        assert hist == gold[f"{key}_hist"]
        u_ref = np.load(os.path.join(GOLD, f"config1_{key}_u.npy"))
        assert np.array_equal(x, u_ref)
        sig = X.homogenized_stress(rho, c, h, x, eb, (1.0, 1.0))
        assert np.array_equal(sig, np.array(gold[f"{key}_sigma"]))


# ---------------------------------------------------------------------------
# 3-D: first-principles pins
# ---------------------------------------------------------------------------

def kuhn_tets():
    """Vertices (relative lattice offsets) of the d! simplices of a voxel,
    independently of oracle.edge_offsets: the monotone path from the corner
    x + e0 that steps -e0 along axis 0 and +e_j along the others, in the
    order of permutation pi."""
    out = []
    for perm in itertools.permutations(range(3)):
        v = np.array([1, 0, 0])
        verts = [v.copy()]
        for a in perm:
            v = v.copy()
            v[a] += -1 if a == 0 else 1
            verts.append(v)
        out.append(verts)
    return out


def dense_k3(n, rho, lam, mu, h):
    """Dense K = sum over voxels/tets of rho w B^T C B with P1 gradients from
    the inverse of the vertex-coordinate matrix (no finite differences)."""
    N = n ** 3
    c = X.isotropic_stiffness(3, lam, mu)
    K = np.zeros((3 * N, 3 * N))
    vol = h[0] * h[1] * h[2] / 6.0
    pairs = X.mandel_pairs(3)
    for x0, x1, x2 in itertools.product(range(n), repeat=3):
        for verts in kuhn_tets():
            P = np.array([[1.0] + [verts[k][a] * h[a] for a in range(3)] for k in range(4)])
            coef = np.linalg.inv(P)  # column k: coefficients of shape fn k
            grads = coef[1:, :].T     # (4 vertices, 3 directions)
            nodes = [((x0 + v[0]) % n) * n * n + ((x1 + v[1]) % n) * n + (x2 + v[2]) % n
                     for v in verts]
            B = np.zeros((6, 12))
            for k in range(4):
                for m, (i, j) in enumerate(pairs):
                    if i == j:
                        B[m, 3 * k + i] += grads[k][i]
                    else:
                        B[m, 3 * k + i] += grads[k][j] / math.sqrt(2)
                        B[m, 3 * k + j] += grads[k][i] / math.sqrt(2)
            Ke = rho[x0, x1, x2] * vol * B.T @ c @ B
            dofs = [a * N + nodes[k] for k in range(4) for a in range(3)]
            # dofs ordering above is (k, a); B columns are 3k + a
            for p in range(12):
                for q in range(12):
                    K[dofs[p], dofs[q]] += Ke[p, q]
    return K


def test_oracle_3d_matches_dense_assembly():
    rng = np.random.default_rng(0)
    n = 3
    h = (0.4, 0.3, 0.5)
    rho = rng.uniform(0.1, 2.0, (n, n, n))
    lam, mu = 0.7, 0.45
    K = dense_k3(n, rho, lam, mu, h)
    c = X.isotropic_stiffness(3, lam, mu)
    for _ in range(3):
        u = rng.normal(size=(3, n, n, n))
        ours = X.apply_K(rho, c, h, u).reshape(-1)
        ref = K @ u.reshape(-1)
        assert np.abs(ours - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.abs(K - K.T).max() <= 1e-12 * np.abs(K).max()


def test_oracle_3d_known_answers():
    rng = np.random.default_rng(1)
    n = (8, 8, 8)
    lam, mu = 2.0 / 3.0, 0.5
    c = X.isotropic_stiffness(3, lam, mu)
    h = X.pixel_size(n, (1.0, 1.0, 1.0))
    rho = rng.uniform(0.05, 2.0, n)
    t = np.ones((3,) + n) * np.array([1.3, -0.7, 0.2])[:, None, None, None]
    assert np.abs(X.apply_K(rho, c, h, t)).max() == 0.0          # rigid translations
    eb = rng.normal(size=6)
    sig = X.homogenized_stress(np.ones(n), c, h, np.zeros((3,) + n), eb, (1.0,) * 3)
    assert np.allclose(sig, c @ eb, rtol=0, atol=1e-13)            # uniform medium
    blocks = X.assemble_green(n, (1.0,) * 3, c)
    assert np.abs(blocks[0, 0, 0]).max() == 0.0
    u = rng.normal(size=(3,) + n)
    gk = X.apply_green(blocks, X.apply_K(np.ones(n), c, h, u))
    assert np.abs(gk - (u - u.mean(axis=(1, 2, 3))[:, None, None, None])).max() <= 1e-12
    # laminate closed form: rho = rho(i0)
    r1 = rng.uniform(1e-3, 1.0, n[0])
    rho_l = np.broadcast_to(r1[:, None, None], n).copy()
    H = 1.0 / np.mean(1.0 / (r1 * (lam + 2 * mu)))
    for e, expect in ((np.array([1.0, 0, 0, 0, 0, 0]), np.array([H, H * lam / (lam + 2 * mu),
                                                                 H * lam / (lam + 2 * mu), 0, 0, 0])),
                      (np.array([0, 0, 0, 0, 0, 1.0]), np.array([0, 0, 0, 0, 0,
                                                                 2 * mu / np.mean(1 / r1)]))):
        f = X.assemble_rhs(rho_l, c, h, e)
        it, hist, term, x = X.pcg(rho_l, c, h, f, "green", blocks, eta=1e-26, max_iter=200)
        s = X.homogenized_stress(rho_l, c, h, x, e, (1.0,) * 3)
        assert np.abs(s - expect).max() <= 1e-12 * np.abs(expect).max()


def test_oracle_jacobi_equals_impulse_diagonal_3d():
    rng = np.random.default_rng(2)
    n = (4, 4, 4)
    c = X.isotropic_stiffness(3, 2.0 / 3.0, 0.5)
    h = X.pixel_size(n, (1.0, 1.0, 1.0))
    rho = rng.uniform(0.1, 2.0, n)
    inv = X.assemble_jacobi(rho, c, h)
    diag = np.empty((3,) + n)
    for a in range(3):
        for idx in np.ndindex(*n):
            e = np.zeros((3,) + n)
            e[(a,) + idx] = 1.0
            diag[(a,) + idx] = X.apply_K(rho, c, h, e)[(a,) + idx]
    assert np.abs(inv - 1.0 / np.sqrt(diag)).max() <= 1e-14 * inv.max()


def test_generator_matches_reference_recipe():
    """The 2-D input generator reproduces the reference's own filter +
    rescale pipeline (microstructures.py:73-115) bit for bit."""
    ref = os.path.join("/root/reference", "pkg", "src")
    if not os.path.isdir(ref):
        pytest.skip("reference not mounted (GPU box)")
    import sys
    sys.path.insert(0, ref)
    from jfft import grid as RG, microstructures as RM
    from paper_2508_02613_b200 import microstructures as ms
    rng = np.random.default_rng(3)
    v = (rng.random((32, 32)) < 0.5).astype(float)
    f = RG.ScalarField(RG.make_grid(32), v)
    for _ in range(4):
        f = RM.gaussian_filter(f)
    f = RM.rescale_contrast(f, 1e4)
    assert np.array_equal(ms.bernoulli_smoothed(32, 4, 1e4, 3), f.values)


def test_load_case_pairings_match_reference():
    """oracle.strain_pairings / stress_matrix restate topopt.py:130-141; pinned
    against the reference's own functions on random 2-D load solutions."""
    ref = os.path.join("/root/reference", "pkg", "src")
    if not os.path.isdir(ref):
        pytest.skip("reference not mounted (GPU box)")
    import sys
    import types
    sys.path.insert(0, ref)
    from jfft import grid as RG, material as RMat, operators as RO, topopt as RT
    rng = np.random.default_rng(4)
    n, lengths = 12, (1.0, 1.5)
    grid = RG.make_grid(n, lengths)
    mat = RMat.isotropic_material(0.6, 0.35)
    rho = rng.uniform(0.1, 1.0, (n, n))
    us = rng.normal(size=(3, 2, n, n))
    loads = np.eye(3)
    op = RO.make_operator(RG.ScalarField(grid, rho), mat)
    strains = np.stack([RO.total_strain(op, RG.VectorField(grid, us[g]), loads[g]).values
                        for g in range(3)])
    problem = types.SimpleNamespace(grid=grid, material=mat)
    c = X.isotropic_stiffness(2, 0.6, 0.35)
    h = X.pixel_size((n, n), lengths)
    assert np.allclose(X.strain_pairings(c, h, us, loads), RT._strain_pairings(problem, strains),
                       rtol=1e-13, atol=1e-13)
    assert np.allclose(X.stress_matrix(rho, c, h, us, loads, lengths),
                       RT._stress_matrix(problem, strains, rho), rtol=1e-13, atol=1e-15)
