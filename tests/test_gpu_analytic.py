"""Closed-form checks of the GPU exit law, the analytic oracles of the
reference's own suite run on this library: uniform exits from the disc
centre (T/test_walk.py:60-68), the annulus hit probability ln(R/r)/ln(R/rho)
(T/test_walk.py:70-78, T/test_acceptance.py:113-132) and the 3D concentric
shell hit probability (1/r - 1/R)/(1/rho - 1/R) (T/oracles.py:96-98).

K = I, so both chains step on the inscribed sphere; every precision/chain
pair is checked.  The null probabilities are known exactly, so each check is
an exact two-sided binomial test (scipy.stats.binomtest), Bonferroni-
corrected to a family-wise level of 1e-4 per test, with 1e6 FP32 walks per
case (the reference uses 1e5 at 3 sigma).
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LEVEL = 1e-4
VARIANTS = [("ref64", "woe"), ("fp32", "woe"), ("fp32", "max")]


@pytest.fixture(scope="module")
def B():
    from paper_2409_03686_b200 import _native, backend

    _native.require_device(0)
    return backend


def _binom_two_sided_p(k: int, n: int, p: float) -> float:
    """Exact two-sided binomial p-value (sum of the probabilities of all
    outcomes no more likely than k), via scipy when present."""
    from scipy.stats import binomtest

    return binomtest(k, n, p).pvalue


def _identity(d):
    from paper_2409_03686_b200.conductivity import make_tensor

    return make_tensor(np.eye(d)).k_sqrt


@pytest.mark.parametrize("precision,chain", VARIANTS)
def test_exits_uniform_from_disc_centre(B, precision, chain):
    from paper_2409_03686_b200.geometry import Ball, Domain

    dom = Domain(2, Ball(np.zeros(2), 1.0), (), frozenset({0}))
    n = 10**6 if precision == "fp32" else 2 * 10**5
    x, _, _ = B.run_exits(dom, _identity(2), np.zeros(2), 0, 2024, 1e-6, 10**6, n,
                          precision=precision, chain=chain)
    ang = np.mod(np.arctan2(x[:, 1], x[:, 0]), 2.0 * np.pi)
    counts, _ = np.histogram(ang, bins=16, range=(0.0, 2.0 * np.pi))
    pv = [_binom_two_sided_p(int(c), n, 1.0 / 16) for c in counts]
    assert min(pv) * 16 > LEVEL, (counts, pv)
    assert np.allclose(np.hypot(x[:, 0], x[:, 1]), 1.0, atol=2e-6)


@pytest.mark.parametrize("precision,chain", VARIANTS)
def test_annulus_hit_probability(B, precision, chain):
    from paper_2409_03686_b200.geometry import Ball, Domain

    dom = Domain(2, Ball(np.zeros(2), 1.0), (Ball(np.zeros(2), 0.5),), frozenset({0}))
    n = 10**6 if precision == "fp32" else 2 * 10**5
    for r0 in (0.95, 0.7):
        _, _, comp = B.run_exits(dom, _identity(2), np.array([r0, 0.0]), 3, 77, 1e-6, 10**6, n,
                                 precision=precision, chain=chain)
        p = math.log(1.0 / r0) / math.log(1.0 / 0.5)
        k = int(np.count_nonzero(comp == 1))
        assert _binom_two_sided_p(k, n, p) * 2 > LEVEL, (r0, k / n, p)


@pytest.mark.parametrize("precision,chain", VARIANTS)
def test_shell3d_hit_probability(B, precision, chain):
    from paper_2409_03686_b200.geometry import Ball, Domain

    dom = Domain(3, Ball(np.zeros(3), 1.0), (Ball(np.zeros(3), 0.5),), frozenset({0}))
    n = 10**6 if precision == "fp32" else 10**5
    for r0 in (0.9, 0.6):
        start = np.array([0.0, r0 * 0.6, r0 * 0.8])
        _, _, comp = B.run_exits(dom, _identity(3), start, 5, 91, 1e-6, 10**6, n,
                                 precision=precision, chain=chain)
        p = (1.0 / r0 - 1.0) / (1.0 / 0.5 - 1.0)
        k = int(np.count_nonzero(comp == 1))
        assert _binom_two_sided_p(k, n, p) * 2 > LEVEL, (r0, k / n, p)
