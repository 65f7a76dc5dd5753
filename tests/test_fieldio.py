"""Field file format (grid.py:218-295) against files written by the
reference's own save_field (tests/golden/fields, made by make_fields.py),
plus 3-D round trips and the reference's validation errors.  The device
load/save paths are in test_gpu_fieldio.py."""

import json
import os

import numpy as np
import pytest

from paper_2508_02613_b200 import fieldio as F
from paper_2508_02613_b200 import grid as G

FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fields")


@pytest.mark.parametrize("kind,cls", [("scalar", G.ScalarField), ("vector", G.VectorField),
                                      ("quad", G.QuadField)])
def test_reads_reference_files(kind, cls):
    f = F.load_field(os.path.join(FIX, kind))
    assert type(f) is cls
    assert f.grid == G.make_grid(6, (1.0, 2.0))
    assert np.array_equal(f.values, np.load(os.path.join(FIX, "values.npz"))[kind])


@pytest.mark.parametrize("kind", ["scalar", "vector", "quad"])
def test_writes_reference_bytes(tmp_path, kind):
    f = F.load_field(os.path.join(FIX, kind))
    F.save_field(tmp_path / kind, f)
    for ext in (".raw", ".json"):
        ours = open(str(tmp_path / kind) + ext, "rb").read()
        ref = open(os.path.join(FIX, kind) + ext, "rb").read()
        assert ours == ref, ext


@pytest.mark.parametrize("make", [
    lambda g, r: G.ScalarField(g, r.uniform(0.0, 2.0, g.shape)),
    lambda g, r: G.VectorField(g, r.normal(size=(3,) + g.shape)),
    lambda g, r: G.QuadField(g, r.normal(size=(6, 6) + g.shape)),
])
def test_round_trip_3d(tmp_path, make):
    rng = np.random.default_rng(1)
    grid = G.make_grid(5, (1.0, 2.0, 0.5))
    f = make(grid, rng)
    F.save_field(tmp_path / "f", f)
    g = F.load_field(tmp_path / "f")
    assert type(g) is type(f) and g.grid == grid
    assert np.array_equal(g.values, f.values)
    assert json.load(open(str(tmp_path / "f") + ".json"))["d"] == 3
    # x1-fastest: the first raw values run along axis 0
    raw = np.fromfile(str(tmp_path / "f") + ".raw", dtype="<f8")
    first = f.values if f.values.ndim == 3 else f.values.reshape((-1,) + grid.shape)[0]
    assert np.array_equal(raw[:5], first[:, 0, 0])


def test_validation_errors(tmp_path):
    grid = G.make_grid(4)
    F.save_field(tmp_path / "rho", G.ScalarField.full(grid, 1.0))
    hdr = json.load(open(str(tmp_path / "rho") + ".json"))
    for key, val in (("order", "x2-fastest"), ("dtype", "float32"), ("kind", "tensor"),
                     ("d", 4)):
        bad = dict(hdr, **{key: val})
        json.dump(bad, open(str(tmp_path / "bad") + ".json", "w"))
        np.zeros(16).tofile(str(tmp_path / "bad") + ".raw")
        with pytest.raises(ValueError):
            F.load_field(tmp_path / "bad")
    missing = {k: v for k, v in hdr.items() if k != "lengths"}
    json.dump(missing, open(str(tmp_path / "bad") + ".json", "w"))
    with pytest.raises(ValueError):
        F.load_field(tmp_path / "bad")
    np.zeros(15).tofile(str(tmp_path / "rho") + ".raw")
    with pytest.raises(ValueError):
        F.load_field(tmp_path / "rho")
    with pytest.raises(TypeError):
        F.save_field(tmp_path / "x", np.zeros((4, 4)))
