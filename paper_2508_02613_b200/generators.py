"""Device input generators.

The reference's microstructure post-processing (microstructures.py:73-115)
with its own signatures, running in libjfftb200.so (csrc/generators.cu):

* ``gaussian_filter(rho)``            microstructures.py:73-82 (one periodic
  binomial pass per axis; bit-identical to the NumPy rounding order)
* ``threshold(rho_smooth, chi_tot)``  microstructures.py:94-101
* ``rescale_contrast(rho, chi_tot)``  microstructures.py:104-115
* ``total_contrast(rho)``             microstructures.py:85-91

They accept and return ``ScalarField`` objects of the caller's classes (the
reference's or this package's).  For bench-size grids the in-place device
forms work on torch CUDA tensors without a host round trip:
``filter_(t, passes)``, ``rescale_(t, chi)``, ``threshold_(t, chi)``,
``simp_projection_(t, beta, emin)``, and the BASELINE config-5 generator
``simp_density_device`` (seeded uniform noise -> 8 binomial passes ->
tanh(beta (rho - 1/2)) -> min-max -> E = emin + rho^3).
"""

from __future__ import annotations

import ctypes as C
import sys

import numpy as np

from . import _native as N


def _handle_for(grid_or_shape, lengths=None) -> N.GridHandle:
    if hasattr(grid_or_shape, "lengths"):
        d = len(grid_or_shape.lengths)
        return N.grid_handle(d, (grid_or_shape.n,) * d, grid_or_shape.lengths)
    shape = tuple(int(k) for k in grid_or_shape)
    return N.grid_handle(len(shape), shape, lengths or (1.0,) * len(shape))


def _scalar_like(rho, values):
    cls = sys.modules[type(rho).__module__].ScalarField
    site = getattr(rho, "site", "pixel")
    try:
        return cls(rho.grid, values, site=site)
    except TypeError:
        return cls(rho.grid, values)


def _host_call(fn, rho, *args):
    vals = np.array(rho.values, dtype=np.float64, order="C", copy=True)
    N.check(fn(_handle_for(rho.grid).ptr, N.vptr(vals), *args, N.HOST))
    return vals


def gaussian_filter(rho):
    """microstructures.py:73-82: one periodic pass of the separable binomial
    kernel ([1 2 1]/4 along every axis)."""
    return _scalar_like(rho, _host_call(N.load().jfftb_binomial_filter, rho, 1))


def threshold(rho_smooth, chi_tot: float):
    """microstructures.py:94-101: 1 where ``rho_smooth >= 0.5``, else 1/chi."""
    chi = float(chi_tot)
    if chi < 1.0:
        raise ValueError(f"total phase contrast must be >= 1, got {chi}")
    return _scalar_like(rho_smooth,
                        _host_call(N.load().jfftb_threshold, rho_smooth, C.c_double(chi)))


def rescale_contrast(rho, chi_tot: float):
    """microstructures.py:104-115: affine map onto ``[1/chi_tot, 1]``."""
    chi = float(chi_tot)
    if chi < 1.0:
        raise ValueError(f"total phase contrast must be >= 1, got {chi}")
    return _scalar_like(rho, _host_call(N.load().jfftb_rescale_contrast, rho, C.c_double(chi)))


def field_minmax(values, grid=None) -> tuple:
    """(min, max) of a host array or a CUDA tensor (deterministic)."""
    out = np.zeros(2)
    if hasattr(values, "data_ptr"):
        import torch
        torch.cuda.current_stream(values.device).synchronize()
        h = _handle_for(tuple(values.shape))
        N.check(N.load().jfftb_field_minmax(h.ptr, C.c_void_p(values.data_ptr()), N.dptr(out),
                                            N.DEVICE))
    else:
        arr = np.ascontiguousarray(values, dtype=np.float64)
        h = _handle_for(grid) if grid is not None else _handle_for(arr.shape)
        N.check(N.load().jfftb_field_minmax(h.ptr, N.vptr(arr), N.dptr(out), N.HOST))
    return float(out[0]), float(out[1])


def total_contrast(rho) -> float:
    """microstructures.py:85-91: max / min; infinite when voids exist."""
    lo, hi = field_minmax(rho.values, rho.grid)
    if lo < 0.0:
        raise ValueError("negative density")
    return np.inf if lo == 0.0 else hi / lo


# ---- in-place device forms (torch CUDA tensors, C-contiguous float64) ------

def _dev_call(fn, t, *args):
    """Run ``fn(grid, ptr, *args, DEVICE)`` on a tensor: ordered after the
    torch work that produced it and complete before torch touches it again."""
    import torch
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError("expected a contiguous float64 CUDA tensor")
    h = _handle_for(tuple(t.shape))
    torch.cuda.current_stream(t.device).synchronize()
    N.check(fn(h.ptr, C.c_void_p(t.data_ptr()), *args, N.DEVICE))
    N.check(N.load().jfftb_grid_synchronize(h.ptr))
    return t


def filter_(t, passes: int = 1):
    """``passes`` binomial-filter passes of a scalar field tensor, in place."""
    return _dev_call(N.load().jfftb_binomial_filter, t, int(passes))


def rescale_(t, chi: float):
    if float(chi) < 1.0:
        raise ValueError(f"total phase contrast must be >= 1, got {chi}")
    return _dev_call(N.load().jfftb_rescale_contrast, t, C.c_double(float(chi)))


def threshold_(t, chi: float):
    if float(chi) < 1.0:
        raise ValueError(f"total phase contrast must be >= 1, got {chi}")
    return _dev_call(N.load().jfftb_threshold, t, C.c_double(float(chi)))


def simp_projection_(t, beta: float = 8.0, emin: float = 1e-6):
    return _dev_call(N.load().jfftb_simp_projection, t, C.c_double(float(beta)),
                     C.c_double(float(emin)))


def bernoulli_smoothed_device(n: int, filters: int, chi: float = 1e4, seed: int = 0,
                              d: int = 2, device="cuda"):
    """Configs 1-2 on the device: the same seeded Bernoulli(0.5) draw as
    ``microstructures.bernoulli_smoothed`` (host RNG), filtered and rescaled
    in device memory -- bit-identical to the host recipe."""
    import torch
    rng = np.random.default_rng(seed)
    v = (rng.random((n,) * d) < 0.5).astype(float)
    t = torch.from_numpy(v).to(device)
    filter_(t, filters)
    return rescale_(t, chi)


def simp_density_device(n: int = 1024, filters: int = 8, beta: float = 8.0,
                        emin: float = 1e-6, seed: int = 0, device="cuda"):
    """BASELINE config 5 on the device (see ``microstructures.simp_density``
    for the host recipe it reproduces)."""
    import torch
    rng = np.random.default_rng(seed)
    t = torch.from_numpy(rng.random((n,) * 3)).to(device)
    filter_(t, filters)
    return simp_projection_(t, beta, emin)


def _bench(n_dev: int = 1024, n_host: int = 256, filters: int = 8):  # pragma: no cover
    """Time the config-5 post-processing (``filters`` binomial passes + SIMP
    projection) on the device at ``n_dev``^3 against the NumPy host recipe at
    ``n_host``^3; prints one JSON line.  Random draw and upload excluded."""
    import json
    import time

    import torch
    from . import microstructures as ms
    rng = np.random.default_rng(0)
    t = torch.from_numpy(rng.random((n_dev,) * 3)).cuda()
    filter_(t, 1)  # grid context + warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    filter_(t, filters)
    simp_projection_(t, 8.0, 1e-6)
    torch.cuda.synchronize()
    dev_s = time.perf_counter() - t0
    vox = float(n_dev) ** 3
    # per filter pass: one read + one write of the field per axis
    gbps = filters * 3 * 2 * 8 * vox / dev_s / 1e9
    v = rng.random((n_host,) * 3)
    t0 = time.perf_counter()
    for _ in range(filters):
        v = ms.binomial_filter(v)
    v = np.tanh(8.0 * (v - 0.5))
    v = (v - v.min()) / (v.max() - v.min())
    v = 1e-6 + v * v * v
    host_s = time.perf_counter() - t0
    print(json.dumps({"what": "config-5 density post-processing (8 binomial passes + SIMP)",
                      "device_n": n_dev, "device_s": dev_s,
                      "device_Gvox_per_s": vox / dev_s / 1e9, "device_filter_GBps_lower_bound": gbps,
                      "host_n": n_host, "host_s": host_s,
                      "host_Gvox_per_s": float(n_host) ** 3 / host_s / 1e9,
                      "host_cores": 1}))


if __name__ == "__main__":  # pragma: no cover
    _bench()
