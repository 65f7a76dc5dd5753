"""Device field-file paths: the raw payload uploaded as-is and reordered by
jfftb_field_layout must equal the host loader bit for bit, and a device save
must write the same bytes as the host save."""

import os

import numpy as np
import pytest

from paper_2508_02613_b200 import fieldio as F
from paper_2508_02613_b200 import grid as G

pytestmark = pytest.mark.gpu
FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fields")


@pytest.mark.parametrize("kind", ["scalar", "vector", "quad"])
def test_device_load_reference_files(kind):
    k, grid, t = F.load_field_device(os.path.join(FIX, kind))
    assert k == kind and grid == G.make_grid(6, (1.0, 2.0))
    assert np.array_equal(t.cpu().numpy(), F.load_field(os.path.join(FIX, kind)).values)


@pytest.mark.parametrize("n,d,kind", [(33, 3, "vector"), (64, 3, "scalar"), (40, 2, "quad"),
                                      (128, 3, "vector")])
def test_device_round_trip(tmp_path, n, d, kind):
    import torch
    rng = np.random.default_rng(n + d)
    grid = G.make_grid(n, (1.0,) * d)
    lead = {"scalar": (), "vector": (d,), "quad": (G.mandel_dim(d), 2 if d == 2 else 6)}[kind]
    vals = rng.normal(size=lead + (n,) * d)
    cls = {"scalar": G.ScalarField, "vector": G.VectorField, "quad": G.QuadField}[kind]
    F.save_field(tmp_path / "host", cls(grid, vals))
    F.save_field_device(tmp_path / "dev", kind, grid, torch.from_numpy(vals).cuda())
    for ext in (".raw", ".json"):
        assert open(str(tmp_path / "host") + ext, "rb").read() == \
            open(str(tmp_path / "dev") + ext, "rb").read()
    _, _, t = F.load_field_device(tmp_path / "host")
    assert np.array_equal(t.cpu().numpy(), vals)
