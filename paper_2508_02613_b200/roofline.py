"""Algorithmic byte model of one PCG iteration.

"Fused minimum": U = 8 N bytes (one fp64 scalar field); each FFT counts one
read plus one write of its data; a half spectrum of one component counts as
U; the Green blocks are counted as recomputed (0 bytes); halos are free.

    green-jacobi  (18 d + 1) U      green  (14 d + 1) U
    jacobi        (16 d + 1) U      none   (16 d + 1) U

Per-kernel algorithmic bytes (what each of this build's kernels must move at
minimum for its own inputs/outputs) are given by ``kernel_bytes``.
"""

from __future__ import annotations

PER_ITER_U = {"green-jacobi": lambda d: 18 * d + 1, "green": lambda d: 14 * d + 1,
              "jacobi": lambda d: 16 * d + 1, "none": lambda d: 16 * d + 1}

#: stage names of the device profile (jfftb_profile_read order)
STAGES = ("stencil", "alpha", "update", "fft_fwd", "spectral", "finalize", "fft_inv", "pupdate")


def algorithmic_bytes(kind: str, d: int, n_nodes: int) -> int:
    return PER_ITER_U[kind](d) * 8 * int(n_nodes)


def kernel_bytes(stage: str, kind: str, d: int, n_nodes: int, fused: bool = True) -> int:
    """Compulsory bytes of one launch of a stage of this build's iteration
    (stored Green blocks: d = 2 -> 4, d = 3 -> 9 doubles per frequency).

    ``fused`` = the fused-FFT path of power-of-two grids (fused.cu), where
    "update" is pass A (r' = r - alpha Kp and the axis-0 transforms), the
    FFT stages are passes B / B', "spectral" is pass C and "pupdate" is pass I
    (which also carries the lagged x += alpha p)."""
    U = 8 * int(n_nodes)
    gj = kind == "green-jacobi"
    green_planes = 4 if d == 2 else 9
    if stage == "stencil":
        return (2 * d + 1) * U                       # p, rho -> Kp
    if fused and kind in ("green", "green-jacobi"):
        if stage == "update":                        # r, Kp (, D) -> r', spectra
            return (6 * d if gj else 4 * d) * U
        if stage == "pupdate":                       # z^, (D), p, x -> p, x
            return (6 * d if gj else 5 * d) * U
    if stage == "update":
        extra = d if gj else (d if kind == "jacobi" else 0)
        dinv = d if kind in ("jacobi", "green-jacobi") else 0
        return (6 * d + extra + dinv) * U            # x, r, p, Kp -> x, r (+ s / z)
    if stage == "fft_fwd":
        comps = 2 * d if gj else d
        return 2 * comps * U                         # real in, half spectrum out
    if stage == "spectral":
        if kind in ("none", "jacobi"):
            return d * U + green_planes * U // 2
        reads = (2 * d if gj else d) * U
        return reads + d * U + green_planes * U // 2   # spectra in, z^ out, blocks
    if stage == "fft_inv":
        return 2 * d * U if kind in ("green", "green-jacobi") else 0
    if stage == "pupdate":
        return (4 * d if gj else 3 * d) * U          # z', (D), p -> p
    return 0
