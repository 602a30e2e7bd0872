"""Config 5 (spectral-gap sweep): Monte-Carlo consensus on the GPU vs the
reference's values frozen in tests/golden/spectral.npz."""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import spectral_golden
from paper_2002_01119_b200 import spectral

pytestmark = pytest.mark.gpu


def test_monte_carlo_frobenius_matches_reference():
    z = spectral_golden()
    mc = spectral.monte_carlo_consensus(8, 6, 40, seed=2, norm_kind="frobenius")
    assert np.allclose(mc.distances, z["mc8_frob_dist"], rtol=1e-12, atol=1e-15)
    assert np.allclose(mc.halfwidths, z["mc8_frob_half"], rtol=1e-9, atol=1e-15)
    assert np.allclose(mc.squared_distances, z["mc8_frob_sq"], rtol=1e-12, atol=1e-15)


def test_monte_carlo_spectral_matches_reference():
    z = spectral_golden()
    mc = spectral.monte_carlo_consensus(12, 4, 20, seed=3, norm_kind="spectral")
    assert np.allclose(mc.distances, z["mc12_spec_dist"], rtol=1e-10, atol=1e-13)
    assert np.allclose(mc.halfwidths, z["mc12_spec_half"], rtol=1e-7, atol=1e-13)


@pytest.mark.parametrize("L", [8, 16, 32, 64, 128])
def test_randomized_rate_matches_closed_form(L):
    # acceptance criterion pattern (reference test_acceptance.py:108-141): the MC
    # mean of ||prod - U||_F^2 is within 3 standard errors of (L-1) a^k
    mc = spectral.monte_carlo_consensus(L, 5, 1000, seed=2, norm_kind="frobenius")
    se = mc.squared_halfwidths / 1.959963984540054
    for k in range(5):
        exact = spectral.randomized_frobenius_expectation(L, k + 1)
        assert abs(mc.squared_distances[k] - exact) <= 3 * se[k] + 1e-12
