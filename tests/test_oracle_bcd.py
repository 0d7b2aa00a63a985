"""Pins of the oracle's projected block-coordinate filter update (PAPER.md
P:313-317; readings B1-B4), independent of the oracle:
  * K = 1 with a single interior impulse code: Z is an embedding, so the exact block minimiser is the
    s x s crop of the image under the impulse, projected on the unit ball when its norm exceeds 1;
  * with the constraint inactive, repeated sweeps converge to the unconstrained least-squares filters
    computed by numpy.linalg.lstsq on the dense Z matrix (tests/_dense.py), and every sweep lowers
    the fit;
  * a filter whose codes are all zero is left unchanged and flagged.
"""
import numpy as np
import pytest

import oracle
from synth import random_problem
from tests._dense import dense_Z


def _fit(x, d, z):
    return oracle.objective(x, d, z, 0.0, dtype=np.float64)[1]


@pytest.mark.parametrize("scale", [0.05, 3.0])
def test_bcd_single_impulse_is_the_image_crop(scale):
    s, H, W = 5, 12, 11
    P = s - 1
    rng = np.random.default_rng(8)
    x = rng.standard_normal((1, H, W)) * scale
    z = np.zeros((1, 1, H + P, W + P))
    u0, v0 = 7, 6  # footprint rows u0-P..u0, cols v0-P..v0 inside the image
    z[0, 0, u0, v0] = 1.0
    d = rng.standard_normal((1, s, s))
    dn, flags = oracle.filter_step_bcd(x, d, z, dtype=np.float64)
    crop = x[0, u0 - P:u0 + 1, v0 - P:v0 + 1]
    expect = crop / max(1.0, np.linalg.norm(crop))
    assert flags[0] == 0
    assert np.allclose(dn[0], expect, rtol=0, atol=1e-9 * max(1.0, np.abs(expect).max()))


def test_bcd_sweeps_reach_least_squares_when_unconstrained():
    x, d, z = random_problem(12, 2, 3, 3, 9, 8, code_density=0.5)
    x = x.astype(np.float64) * 0.02  # small images -> least-squares filters inside the unit ball
    d = d.astype(np.float64) * 0.1
    z = z.astype(np.float64)
    Z = np.concatenate([dense_Z(z[n], 3) for n in range(2)], axis=0)
    d_ls = np.linalg.lstsq(Z, x.reshape(-1), rcond=None)[0]
    assert np.linalg.norm(d_ls.reshape(3, -1), axis=1).max() < 1.0
    f_prev = _fit(x, d, z)
    dd = d
    for _ in range(60):
        dd, flags = oracle.filter_step_bcd(x, dd, z, sweeps=5, dtype=np.float64)
        f = _fit(x, dd, z)
        assert f <= f_prev * (1 + 1e-12)
        f_prev = f
    assert not flags.any()
    assert np.linalg.norm(dd.ravel() - d_ls) <= 1e-6 * np.linalg.norm(d_ls)


def test_bcd_zero_codes_leave_filter_unchanged():
    x, d, z = random_problem(13, 1, 3, 5, 10, 10, code_density=0.4)
    z[:, 1] = 0.0
    dn, flags = oracle.filter_step_bcd(x, d, z)
    assert list(flags) == [0, 1, 0]
    assert np.array_equal(dn[1], d[1])
    assert (np.linalg.norm(dn.reshape(3, -1), axis=1) <= 1 + 1e-6).all()
