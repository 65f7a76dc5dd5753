"""Field file format on and off the device (grid.py:218-295).

``<base>.json`` header (kind, d, n, lengths, order = "x1-fastest",
dtype = "float64-le") and ``<base>.raw`` payload of little-endian doubles,
planes component-major (Mandel-major then simplex-major for quadrature
fields), each plane in x1-fastest order -- the Fortran order of the
``n x ... x n`` array.  ``save_field`` / ``load_field`` keep the reference's
signatures and write byte-identical files for 2-D fields; they are
d-generic, so 3-D fields use the same format with ``"d": 3``.

``load_field_device`` / ``save_field_device`` move 512^3 / 1024^3 payloads
between a file and a device tensor without a host-side transpose: the raw
bytes are uploaded as they are and reordered by the library's tiled
axis-swap kernel (``jfftb_field_layout``).
"""

from __future__ import annotations

import ctypes as C
import json
import math

import numpy as np

from . import _native as N
from . import grid as G

_KINDS = ("scalar", "vector", "quad")


def _kind_of(field) -> str:
    name = type(field).__name__
    kind = {"ScalarField": "scalar", "VectorField": "vector", "QuadField": "quad"}.get(name)
    if kind is None:
        raise TypeError(f"not a field: {name}")
    return kind


def _nplanes(kind: str, d: int) -> int:
    return {"scalar": 1, "vector": d, "quad": G.mandel_dim(d) * math.factorial(d)}[kind]


def _header(kind: str, grid) -> dict:
    return {"kind": kind, "d": len(grid.lengths), "n": grid.n,
            "lengths": list(grid.lengths), "order": "x1-fastest", "dtype": "float64-le"}


def _write_header(base: str, header: dict) -> None:
    with open(base + ".json", "w") as fh:
        json.dump(header, fh, indent=2)
        fh.write("\n")


def save_field(basepath, field) -> None:
    """grid.py:238-252: write ``<basepath>.json`` and ``<basepath>.raw``."""
    base = str(basepath)
    kind = _kind_of(field)
    grid = field.grid
    d = len(grid.lengths)
    _write_header(base, _header(kind, grid))
    planes = np.asarray(field.values).reshape((_nplanes(kind, d),) + (grid.n,) * d)
    payload = np.concatenate([p.ravel(order="F") for p in planes])
    payload.astype("<f8").tofile(base + ".raw")


def read_header(basepath) -> dict:
    base = str(basepath)
    with open(base + ".json") as fh:
        header = json.load(fh)
    for key in ("kind", "d", "n", "lengths", "order", "dtype"):
        if key not in header:
            raise ValueError(f"field header {base}.json misses key {key!r}")
    if header["d"] not in (2, 3):
        raise ValueError(f"unsupported dimension d={header['d']}")
    if header["order"] != "x1-fastest" or header["dtype"] != "float64-le":
        raise ValueError("unsupported field file layout "
                         f"(order={header['order']!r}, dtype={header['dtype']!r})")
    if header["kind"] not in _KINDS:
        raise ValueError(f"unknown field kind {header['kind']!r}")
    if len(header["lengths"]) != header["d"]:
        raise ValueError("header lengths do not match its dimension")
    return header


def _read_raw(base: str, header: dict) -> np.ndarray:
    d, n = header["d"], header["n"]
    raw = np.fromfile(base + ".raw", dtype="<f8")
    expected = _nplanes(header["kind"], d) * n ** d
    if raw.size != expected:
        raise ValueError(f"{base}.raw holds {raw.size} doubles, expected {expected}")
    return raw


def load_field(basepath, module=None):
    """grid.py:255-295: read a field written by :func:`save_field`; scalar
    fields load as pixel-site densities.  ``module`` selects the container
    classes (default: this package's; pass the reference's ``jfft.grid`` to
    get its containers)."""
    base = str(basepath)
    header = read_header(base)
    M = module or G
    grid = M.make_grid(header["n"], tuple(header["lengths"]))
    raw = _read_raw(base, header)
    d, n, kind = header["d"], header["n"], header["kind"]
    pl = n ** d
    planes = [raw[k * pl:(k + 1) * pl].reshape((n,) * d, order="F")
              for k in range(_nplanes(kind, d))]
    if kind == "scalar":
        return M.ScalarField(grid, planes[0], site="pixel")
    if kind == "vector":
        return M.VectorField(grid, np.stack(planes))
    values = np.stack(planes).reshape((G.mandel_dim(d), math.factorial(d)) + (n,) * d)
    return M.QuadField(grid, values)


# ---- device side -------------------------------------------------------------

def load_field_device(basepath, device="cuda"):
    """Read a field file straight into device memory.  Returns
    ``(kind, grid, tensor)`` with the tensor in the containers' C layout
    (``(n,)*d``, ``(d,) + (n,)*d`` or ``(M, d!) + (n,)*d``)."""
    import torch
    base = str(basepath)
    header = read_header(base)
    d, n, kind = header["d"], header["n"], header["kind"]
    grid = G.make_grid(n, tuple(header["lengths"]))
    raw = torch.from_numpy(_read_raw(base, header)).to(device)
    planes = _nplanes(kind, d)
    out = torch.empty_like(raw)
    # the reorder runs on the tensor's own device (not JFFTB_DEVICE)
    h = N.grid_handle(d, (n,) * d, grid.lengths, device=out.device.index)
    torch.cuda.current_stream(out.device).synchronize()
    N.check(N.load().jfftb_field_layout(h.ptr, C.c_void_p(raw.data_ptr()),
                                        C.c_void_p(out.data_ptr()), planes, 1, N.DEVICE))
    lead = {"scalar": (), "vector": (d,), "quad": (G.mandel_dim(d), math.factorial(d))}[kind]
    return kind, grid, out.reshape(lead + (n,) * d)


def save_field_device(basepath, kind: str, grid, tensor) -> None:
    """Write a device tensor in the container layout of ``kind`` as a field
    file (the reorder runs on the device; one host copy of the payload)."""
    import torch
    if kind not in _KINDS:
        raise ValueError(f"unknown field kind {kind!r}")
    d = len(grid.lengths)
    planes = _nplanes(kind, d)
    t = tensor.contiguous()
    if t.dtype != torch.float64 or t.numel() != planes * grid.n ** d:
        raise ValueError("tensor does not hold a float64 field of that kind and grid")
    out = torch.empty_like(t)
    h = N.grid_handle(d, (grid.n,) * d, grid.lengths, device=t.device.index)
    torch.cuda.current_stream(t.device).synchronize()
    N.check(N.load().jfftb_field_layout(h.ptr, C.c_void_p(t.data_ptr()),
                                        C.c_void_p(out.data_ptr()), planes, 0, N.DEVICE))
    base = str(basepath)
    _write_header(base, _header(kind, grid))
    out.cpu().numpy().astype("<f8", copy=False).tofile(base + ".raw")
