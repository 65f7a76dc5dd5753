"""Field files written by the reference's own save_field (grid.py:238-252),
committed as fixtures for paper_2508_02613_b200.fieldio.  Run in the build
container (the reference is mounted at /root/reference):

    python tests/golden/make_fields.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from jfft.grid import QuadField, ScalarField, VectorField, make_grid, save_field  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fields")


def main():
    os.makedirs(HERE, exist_ok=True)
    rng = np.random.default_rng(5)
    grid = make_grid(6, (1.0, 2.0))
    fields = {
        "scalar": ScalarField(grid, rng.uniform(0.0, 2.0, (6, 6))),
        "vector": VectorField(grid, rng.normal(size=(2, 6, 6))),
        "quad": QuadField(grid, rng.normal(size=(3, 2, 6, 6))),
    }
    arrays = {}
    for name, f in fields.items():
        save_field(os.path.join(HERE, name), f)
        arrays[name] = f.values
    np.savez(os.path.join(HERE, "values.npz"), **arrays)


if __name__ == "__main__":
    main()
