"""Device input generators (csrc/generators.cu) against the host recipes.

The host recipes in ``microstructures`` reproduce the reference's own
gaussian_filter / rescale_contrast bit for bit (test_oracle_pins.py
test_generator_matches_reference_recipe, run where the reference is
mounted), so bitwise agreement here is bitwise agreement with the
reference's NumPy rounding order.  SIMP uses tanh, whose device and libm
implementations may differ in the last ulp (amplified up to ~3x by the
min-max normalisation and the cube): held to 2e-15 relative (~9 ulp).
"""

import numpy as np
import pytest

from paper_2508_02613_b200 import generators as GEN
from paper_2508_02613_b200 import grid as G
from paper_2508_02613_b200 import microstructures as ms

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


@pytest.mark.parametrize("shape", [(2, 2), (3, 5), (7, 7), (64, 64), (256, 256),
                                   (2, 3, 4), (5, 5, 5), (32, 16, 8), (64, 64, 64)])
@pytest.mark.parametrize("passes", [1, 3, 10])
def test_binomial_filter_bitwise(shape, passes):
    torch = _torch()
    rng = np.random.default_rng(sum(shape) + passes)
    v = rng.random(shape)
    ref = v
    for _ in range(passes):
        ref = ms.binomial_filter(ref)
    t = torch.from_numpy(v).cuda()
    GEN.filter_(t, passes)
    assert np.array_equal(t.cpu().numpy(), ref)


def test_reference_signature_host_api():
    """ScalarField in, ScalarField out, input untouched (microstructures.py)."""
    rng = np.random.default_rng(5)
    n = 48
    grid = G.make_grid(n)
    v = (rng.random((n, n)) < 0.5).astype(float)
    f = G.ScalarField(grid, v.copy())
    ref = v
    for _ in range(4):
        f = GEN.gaussian_filter(f)
        ref = ms.binomial_filter(ref)
    assert np.array_equal(f.values, ref)
    r = GEN.rescale_contrast(f, 1e4)
    assert np.array_equal(r.values, ms.rescale_contrast(ref, 1e4))
    assert GEN.total_contrast(r) == pytest.approx(1e4, rel=1e-12)
    th = GEN.threshold(f, 1e3)
    assert np.array_equal(th.values, np.where(ref >= 0.5, 1.0, 1e-3))
    assert np.array_equal(GEN.rescale_contrast(f, np.inf).values,
                          ms.rescale_contrast(ref, np.inf))


def test_generator_errors():
    grid = G.make_grid(8)
    const = G.ScalarField(grid, np.full((8, 8), 0.3))
    with pytest.raises(ValueError):
        GEN.rescale_contrast(const, 10.0)
    with pytest.raises(ValueError):
        GEN.rescale_contrast(G.ScalarField(grid, np.random.default_rng(0).random((8, 8))), 0.5)
    with pytest.raises(ValueError):
        GEN.threshold(const, 0.9)
    with pytest.raises(ValueError):
        GEN.total_contrast(G.ScalarField(grid, np.full((8, 8), -1.0)))
    assert GEN.total_contrast(G.ScalarField(grid, np.zeros((8, 8)))) == np.inf


@pytest.mark.parametrize("n,filters", [(64, 5), (256, 10), (512, 20)])
def test_config12_density_on_device_is_bitwise(n, filters):
    """BASELINE configs 1-2 built in device memory == the host recipe."""
    dev = GEN.bernoulli_smoothed_device(n, filters, 1e4, seed=0)
    assert np.array_equal(dev.cpu().numpy(), ms.bernoulli_smoothed(n, filters, 1e4, 0))


def test_config5_simp_density():
    n = 48
    host = ms.simp_density(n, filters=8, beta=8.0, emin=1e-6, seed=2)
    dev = GEN.simp_density_device(n, filters=8, beta=8.0, emin=1e-6, seed=2).cpu().numpy()
    assert np.abs(dev - host).max() <= 2e-15 * np.abs(host).max()
    assert host.min() == pytest.approx(1e-6, abs=1e-15)
    assert host.max() == pytest.approx(1.0 + 1e-6, rel=1e-15)


def test_minmax_device_tensor():
    torch = _torch()
    rng = np.random.default_rng(9)
    v = rng.normal(size=(33, 17, 9))
    lo, hi = GEN.field_minmax(torch.from_numpy(v).cuda())
    assert (lo, hi) == (v.min(), v.max())
