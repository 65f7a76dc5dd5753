"""CPU oracle for the J-FFT PCG hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The shipped path is the CUDA library under
``paper_2508_02613_b200/`` and fails loudly when that library is missing.

It is a NumPy restatement of the reference package ``jfft`` (pure Python on
NumPy, /root/reference/pkg/src/jfft), written dimension-generic so the same
code serves d = 2 (where it reproduces the reference; pinned by
``tests/test_oracle_pins.py`` against fixtures produced by the reference
itself, see ``tests/golden/make_golden.py``) and d = 3 (where the reference
has no implementation; the 3-D discretisation below is this build's choice,
documented in DESIGN.md, and pinned by first-principles known answers:
dense assembly, laminate closed form, uniform-medium stress, G K_ref = I - mean).

Discretisation (d-generic, reduces to the reference for d = 2)
----------------------------------------------------------------
Every voxel with low corner ``x`` is split into d! simplices, one per
permutation ``pi`` of the axes (lexicographic order = simplex index ``t``).
Simplex ``pi`` is the monotone lattice path that starts at ``x + e_0`` and
steps ``-e_0`` along axis 0 and ``+e_j`` along every other axis, in the order
``pi``.  For d = 2 this is exactly the reference's split along the
lower-right to upper-left diagonal (fem.py:3-12): t = 0 is the lower
triangle, t = 1 the upper one.  P1 gradients are constant per simplex; the
column ``a`` of the displacement gradient is the forward difference
``D_a u`` taken on the path edge along axis ``a``, whose low node is
``x + o(pi, a)`` (``edge_offsets``).  One quadrature point per simplex with
weight ``prod(h) / d!`` (fem.py:36-38).

Mandel order: d = 2 (11, 22, sqrt2*12) as grid.py:172-188; d = 3
(11, 22, 33, sqrt2*23, sqrt2*13, sqrt2*12).
"""

from __future__ import annotations

import itertools
import math

import numpy as np

SQRT2 = float(np.sqrt(2.0))

#: Termination defaults (solver.py:27,30).
DEFAULT_ETA_CG = 1e-6
DEFAULT_MAX_ITER = 999
CONVERGED = "converged"
ITERATION_CAP = "iteration-cap"
#: Pseudo-inverse cutoff (preconditioners.py:26).
EIG_CUTOFF = 1e-12
KINDS = ("none", "green", "jacobi", "green-jacobi")


class SolverAbortError(RuntimeError):
    """solver.py:40-41."""


# ---------------------------------------------------------------------------
# index tables
# ---------------------------------------------------------------------------

def mandel_pairs(d: int):
    """Mandel component -> (i, j) tensor index pair."""
    if d == 2:
        return [(0, 0), (1, 1), (0, 1)]
    if d == 3:
        return [(0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1)]
    raise ValueError(f"unsupported dimension {d}")


def mandel_index(d: int, i: int, j: int) -> int:
    for m, (a, b) in enumerate(mandel_pairs(d)):
        if (a, b) == (i, j) or (a, b) == (j, i):
            return m
    raise KeyError((i, j))


def simplices(d: int):
    """Axis permutations in lexicographic order (one simplex each)."""
    return list(itertools.permutations(range(d)))


def edge_offsets(d: int):
    """``o[t][a]``: low node (relative to the voxel corner) of the path edge
    of simplex ``t`` along axis ``a`` (see module docstring).

    d = 2 gives o[0] = ((0,0),(0,0)), o[1] = ((0,1),(1,0)), the anchors of
    fem.py:64-72.
    """
    out = []
    for perm in simplices(d):
        pos = {ax: k for k, ax in enumerate(perm)}
        row = []
        for a in range(d):
            o = []
            for j in range(d):
                if j == a:
                    o.append(0)
                elif j == 0:
                    o.append(0 if pos[j] < pos[a] else 1)
                else:
                    o.append(1 if pos[j] < pos[a] else 0)
            row.append(tuple(o))
        out.append(tuple(row))
    return tuple(out)


def _roll(a: np.ndarray, shift, axes):
    shift = tuple(int(s) for s in shift)
    if not any(shift):
        return a
    return np.roll(a, shift, axis=axes)


# ---------------------------------------------------------------------------
# material (material.py:25-46, generalised to d = 3)
# ---------------------------------------------------------------------------

def isotropic_stiffness(d: int, lam: float, mu: float) -> np.ndarray:
    lam, mu = float(lam), float(mu)
    if mu <= 0.0 or lam + mu <= 0.0:
        raise ValueError(f"stiffness not positive definite (lambda={lam}, mu={mu})")
    m = 3 if d == 2 else 6
    c = np.zeros((m, m))
    for i in range(d):
        for j in range(d):
            c[i, j] = lam
        c[i, i] = lam + 2.0 * mu
    for k in range(d, m):
        c[k, k] = 2.0 * mu
    return c


# ---------------------------------------------------------------------------
# FE kernels (fem.py:41-83, operators.py:43-101)
# ---------------------------------------------------------------------------

def pixel_size(n, lengths):
    return tuple(float(l) / int(k) for l, k in zip(lengths, n))


def sym_gradient(u: np.ndarray, h) -> np.ndarray:
    """(d, *n) nodal field -> (M, d!, *n) Mandel strain per simplex."""
    d = u.shape[0]
    axes = tuple(range(d))
    offs = edge_offsets(d)
    # D_a u_i at every node (fem.py:41-46)
    diff = [[(np.roll(u[i], -1, axis=a) - u[i]) / h[a] for a in range(d)]
            for i in range(d)]
    ntet = len(offs)
    pairs = mandel_pairs(d)
    s = np.empty((len(pairs), ntet) + u.shape[1:])
    for t in range(ntet):
        def g(i, j):
            # d u_i / d x_j on simplex t, read at the edge base x + o(t, j)
            return _roll(diff[i][j], [-k for k in offs[t][j]], axes)
        for m, (i, j) in enumerate(pairs):
            if i == j:
                s[m, t] = g(i, i)
            else:
                s[m, t] = (g(i, j) + g(j, i)) / SQRT2
    return s


def sym_gradient_adjoint(s: np.ndarray, h) -> np.ndarray:
    """Exact transpose of :func:`sym_gradient` (fem.py:76-83)."""
    d = s.ndim - 2
    axes = tuple(range(d))
    offs = edge_offsets(d)
    ntet = len(offs)
    f = np.empty((d,) + s.shape[2:])
    for i in range(d):
        order = [i] + [a for a in range(d) if a != i]
        acc = None
        for a in order:
            m = mandel_index(d, i, a)
            e = s[m, 0]
            e = _roll(e, offs[0][a], axes)
            for t in range(1, ntet):
                e = e + _roll(s[m, t], offs[t][a], axes)
            term = (np.roll(e, 1, axis=a) - e) / h[a]
            if a != i:
                term = term / SQRT2
            acc = term if acc is None else acc + term
        f[i] = acc
    return f


def quad_weight(h) -> float:
    return float(np.prod(h)) / math.factorial(len(h))


def weighted_stress(rho, c, h, eps):
    """W * rho * C0 * eps, fused scale (operators.py:43-48)."""
    sig = np.einsum("mk,k...->m...", c, eps)
    sig *= (quad_weight(h) * rho)[None, None]
    return sig


def apply_K(rho, c, h, u):
    """K(rho) u = B^T W rho C0 B u (operators.py:51-58)."""
    eps = sym_gradient(u, h)
    return sym_gradient_adjoint(weighted_stress(rho, c, h, eps), h)


def assemble_rhs(rho, c, h, eps_bar):
    """f = -B^T W rho C0 E (operators.py:61-76)."""
    eps_bar = np.asarray(eps_bar, dtype=np.float64)
    d = rho.ndim
    m = c.shape[0]
    if eps_bar.shape != (m,):
        raise ValueError(f"macroscopic strain must have shape ({m},)")
    if not np.all(np.isfinite(eps_bar)):
        raise ValueError("macroscopic strain must be finite")
    ntet = math.factorial(d)
    eps = np.broadcast_to(eps_bar.reshape((m, 1) + (1,) * d), (m, ntet) + rho.shape)
    sig = weighted_stress(rho, c, h, eps)
    return -sym_gradient_adjoint(sig, h)


def total_strain(h, u, eps_bar):
    """operators.py:79-83."""
    d = u.shape[0]
    eps = sym_gradient(u, h)
    eps += np.asarray(eps_bar, dtype=np.float64).reshape((-1,) + (1,) * (d + 1))
    return eps


def residual_force(rho, c, h, u, eps_bar):
    """operators.py:86-95."""
    sig = np.einsum("mk,k...->m...", c, total_strain(h, u, eps_bar)) * rho[None, None]
    sig *= quad_weight(h)
    return -sym_gradient_adjoint(sig, h)


def homogenized_stress(rho, c, h, u, eps_bar, lengths):
    """(w/|Y|) sum_Q rho C0 eps (operators.py:98-101, fem.py:106-111)."""
    d = u.shape[0]
    sig = np.einsum("mk,k...->m...", c, total_strain(h, u, eps_bar)) * rho[None, None]
    scale = quad_weight(h) / float(np.prod(lengths))
    return scale * sig.sum(axis=tuple(range(1, d + 2)))


def strain_pairings(c, h, us, loads):
    """topopt.py:130-133 (_strain_pairings), d-generic: for solutions
    ``us[g]`` of loads ``loads[g]``, P[g, c] = sum_t eps_c^T C0 eps_g per pixel."""
    strains = np.stack([total_strain(h, u, e) for u, e in zip(us, loads)])
    c_eps = np.einsum("mk,gkt...->gmt...", c, strains)
    return np.einsum("cmt...,gmt...->gc...", strains, c_eps)


def stress_matrix(rho, c, h, us, loads, lengths):
    """topopt.py:136-141 (_stress_matrix): (w/|Y|) sum_x rho P[g, c]."""
    d = rho.ndim
    P = strain_pairings(c, h, us, loads)
    return quad_weight(h) / float(np.prod(lengths)) * np.einsum(
        "gc" + "xyz"[:d] + "," + "xyz"[:d] + "->gc", P, rho)


# ---------------------------------------------------------------------------
# preconditioners (preconditioners.py:50-136)
# ---------------------------------------------------------------------------

def assemble_green(n, lengths, c_ref) -> np.ndarray:
    """Per-frequency pseudo-inverse blocks, shape (*n[:-1], n[-1]//2+1, d, d)."""
    n = tuple(int(k) for k in n)
    d = len(n)
    h = pixel_size(n, lengths)
    ones = np.ones(n)
    axes = tuple(range(1, d + 1))
    spec = n[:-1] + (n[-1] // 2 + 1,)
    khat = np.empty(spec + (d, d), dtype=np.complex128)
    for beta in range(d):
        imp = np.zeros((d,) + n)
        imp[(beta,) + (0,) * d] = 1.0
        resp = apply_K(ones, c_ref, h, imp)
        khat[..., :, beta] = np.moveaxis(np.fft.rfftn(resp, axes=axes), 0, -1)
    khat[(0,) * d] = 0.0
    khat = 0.5 * (khat + np.conj(np.swapaxes(khat, -1, -2)))
    w, v = np.linalg.eigh(khat)
    cutoff = EIG_CUTOFF * np.clip(w[..., -1:], 0.0, None)
    inv = np.where(w > cutoff, 1.0, 0.0) / np.where(w > cutoff, w, 1.0)
    blocks = np.einsum("...ab,...b,...cb->...ac", v, inv, np.conj(v))
    blocks[(0,) * d] = 0.0
    return blocks


def apply_green(blocks, r):
    d = r.shape[0]
    n = r.shape[1:]
    axes = tuple(range(1, d + 1))
    rhat = np.fft.rfftn(r, axes=axes)
    if d == 2:
        zhat = np.einsum("xyab,bxy->axy", blocks, rhat)
    else:
        zhat = np.einsum("xyzab,bxyz->axyz", blocks, rhat)
    return np.fft.irfftn(zhat, s=n, axes=axes)


def assemble_jacobi(rho, c, h) -> np.ndarray:
    """Comb probing, d * 2^d applications (preconditioners.py:97-119)."""
    d = rho.ndim
    n = rho.shape
    if any(k % 2 for k in n):
        raise ValueError("diagonal probing requires an even node count")
    diag = np.empty((d,) + n)
    for alpha in range(d):
        for offs in itertools.product((0, 1), repeat=d):
            comb = np.zeros((d,) + n)
            sl = (alpha,) + tuple(slice(o, None, 2) for o in offs)
            comb[sl] = 1.0
            resp = apply_K(rho, c, h, comb)
            diag[sl] = resp[sl]
    if np.any(diag < 0.0) or not np.all(np.isfinite(diag)):
        raise ValueError("probed diagonal has negative or non-finite entries")
    diag[diag == 0.0] = 1.0
    return 1.0 / np.sqrt(diag)


def apply_precond(kind, blocks, inv_sqrt, r):
    """Preconditioner.apply (preconditioners.py:156-163)."""
    if kind == "none":
        return r.copy()
    if kind == "green":
        return apply_green(blocks, r)
    if kind == "jacobi":
        return inv_sqrt * (inv_sqrt * r)
    if kind == "green-jacobi":
        return inv_sqrt * apply_green(blocks, inv_sqrt * r)
    raise ValueError(f"unknown preconditioner {kind!r}")


# ---------------------------------------------------------------------------
# PCG (solver.py:64-140)
# ---------------------------------------------------------------------------

def _dot(a, b) -> float:
    return float(np.vdot(a, b))


def pcg(rho, c, h, rhs, kind, blocks, inv_sqrt=None, eta=DEFAULT_ETA_CG,
        max_iter=DEFAULT_MAX_ITER, return_x=True):
    """Returns (iterations, history, terminated, x)."""

    def checked(v, what):
        if not np.isfinite(v):
            raise SolverAbortError(f"{what} became non-finite in PCG")
        return v

    x = np.zeros_like(rhs)
    r = rhs.copy()
    z = apply_precond(kind, blocks, inv_sqrt, r)
    gr = z if kind == "green" else apply_green(blocks, r)
    g2 = checked(_dot(r, gr), "residual Green norm")
    hist = [g2]
    if g2 <= eta:
        return 0, hist, CONVERGED, x
    rz = checked(_dot(r, z), "preconditioned residual product")
    p = z.copy()
    it = 0
    term = ITERATION_CAP
    while it < max_iter:
        kp = apply_K(rho, c, h, p)
        curv = checked(_dot(p, kp), "search-direction curvature")
        if curv <= 0.0:
            raise SolverAbortError(f"non-positive curvature {curv:.3e} in PCG")
        alpha = rz / curv
        x += alpha * p
        r -= alpha * kp
        it += 1
        z = apply_precond(kind, blocks, inv_sqrt, r)
        gr = z if kind == "green" else apply_green(blocks, r)
        g2 = checked(_dot(r, gr), "residual Green norm")
        hist.append(g2)
        if g2 <= eta:
            term = CONVERGED
            break
        rz_new = checked(_dot(r, z), "preconditioned residual product")
        beta = rz_new / rz
        p *= beta
        p += z
        rz = rz_new
    d = rhs.shape[0]
    x -= x.mean(axis=tuple(range(1, d + 1))).reshape((d,) + (1,) * d)
    return it, hist, term, x


# ---------------------------------------------------------------------------
# roofline byte model
# ---------------------------------------------------------------------------

def algorithmic_bytes(kind: str, d: int, n_nodes: int) -> int:
    """Fused-minimum bytes per PCG iteration: (18d+1)U (green-jacobi),
    (14d+1)U (green), (16d+1)U (jacobi / none), U = 8 N."""
    u = 8 * int(n_nodes)
    per = {"green-jacobi": 18 * d + 1, "green": 14 * d + 1,
           "jacobi": 16 * d + 1, "none": 16 * d + 1}[kind]
    return per * u
