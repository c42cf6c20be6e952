"""Input recipe checks (DESIGN.md input recipe; BASELINE.json configs 3 and 4): the seeded RSA
cells have non-overlapping spheres under the periodic minimum image, the requested sphere
count and radius, and a voxelised volume fraction close to phi."""
import math

import numpy as np
import pytest

import synth


@pytest.mark.parametrize("n_spheres, phi, seed", [(30, 0.20, 3), (400, 0.25, 4)])
def test_rsa_non_overlapping_periodic(n_spheres, phi, seed):
    c, r = synth.rsa_centres(n_spheres, phi, seed)
    assert c.shape == (n_spheres, 3)
    assert r == pytest.approx((phi * 3.0 / (4.0 * math.pi * n_spheres)) ** (1.0 / 3.0))
    d = c[:, None, :] - c[None, :, :]
    d -= np.round(d)
    dist = np.sqrt((d ** 2).sum(-1)) + np.eye(n_spheres) * 10.0
    assert dist.min() >= 2.0 * r


def test_config4_cell_matches_recipe():
    cfg = synth.config4(n=64)
    assert cfg.n == (64, 64, 64)
    assert cfg.extra["centres"].shape == (400, 3)
    assert abs(cfg.phases.mean() - 0.25) < 0.01          # voxelised 25 % at 64^3 (512^3: 0.2500)
    c3 = synth.config3(n=64)
    assert cfg.stress_mask == c3.stress_mask and cfg.load_comp == c3.load_comp
    assert np.array_equal(cfg.ell, c3.ell) and cfg.source_phase == c3.source_phase
