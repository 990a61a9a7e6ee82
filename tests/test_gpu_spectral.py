"""Device Gram / SVD / eigendecomposition (spectral.py)
against the reference's host routines (S/estimator.py:112-118 _gram,
S/linalg.py svd / sym_eig, S/tsvd.py), imported from oracle/_ref.

Tolerances: float64 with a different summation order -> entries within
1e-12 of the matrix scale; spectra within 1e-10 relative; reconstructions
(sign-invariant) within 1e-8 relative.  The Gram must be exactly symmetric,
as the reference's mirrored upper triangle is.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref"
need_ref = pytest.mark.skipif(not (REF / "exitmeasure").exists(), reason="oracle/_ref not built")


def _ref():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import exitmeasure

    return exitmeasure


@pytest.fixture(scope="module")
def problem():
    """An A1 of counts/n with the structure of a real run (rows sum < 1,
    sparse-ish, decaying spectrum), 512 poles x 384 cells."""
    from paper_2409_03686_b200 import _native

    _native.require_device(0)
    rng = np.random.default_rng(3686)
    m, m1, n = 512, 384, 10_000
    p = rng.dirichlet(np.full(m1, 0.3), size=m) * rng.uniform(0.3, 0.9, size=(m, 1))
    a1 = rng.binomial(n, p) / n
    sigma1 = rng.uniform(0.5, 1.5, m1) / m1
    nu = rng.uniform(0.5, 1.0, m)
    return a1, sigma1, nu


@need_ref
def test_gram_matches_host(problem):
    from paper_2409_03686_b200 import spectral

    ref = _ref()
    a1, sigma1, nu = problem
    g_ref = ref.estimator._gram(a1, sigma1, nu)
    g = spectral.gram(a1, sigma1, nu)
    assert g.shape == g_ref.shape and g.dtype == np.float64
    assert np.array_equal(g, g.T)
    assert np.max(np.abs(g - g_ref)) <= 1e-12 * np.max(np.abs(g_ref))


def test_gram_from_device_counts(problem):
    """The count rows of a device run feed the Gram without a host copy."""
    import torch

    from paper_2409_03686_b200 import spectral

    a1, sigma1, nu = problem
    n = 10_000
    counts = np.concatenate([np.zeros((a1.shape[0], 7), np.int64),
                             np.rint(a1 * n).astype(np.int64)], axis=1)
    dev = torch.as_tensor(counts, device="cuda")
    g = spectral.gram_from_counts(dev, 7, n, sigma1, nu)
    assert g.is_cuda
    g_host = spectral.gram(counts[:, 7:] / n, sigma1, nu)
    assert np.max(np.abs(g.cpu().numpy() - g_host)) <= 1e-12 * np.max(np.abs(g_host))


@need_ref
def test_svd_and_eig_match_host(problem):
    from paper_2409_03686_b200 import spectral

    ref = _ref()
    a1, sigma1, nu = problem
    m = (nu[:, None] * a1) / np.sqrt(sigma1)[None, :]
    u, s, v = spectral.svd(m)
    u_r, s_r, v_r = ref.linalg.svd(m)
    assert u.shape == u_r.shape and v.shape == v_r.shape
    assert np.allclose(s, s_r, rtol=1e-10, atol=1e-14 * s_r[0])
    k = min(m.shape)
    assert np.allclose((u[:, :k] * s) @ v[:, :k].T, m, atol=1e-12 * s_r[0])
    g = ref.estimator._gram(a1, sigma1, nu)
    w, vec = spectral.sym_eig(g)
    e_r = ref.linalg.sym_eig(g)
    assert np.all(np.diff(w) <= 0)
    assert np.allclose(w, e_r.eigenvalues, rtol=1e-10, atol=1e-13 * e_r.eigenvalues[0])
    assert np.allclose(vec.T @ vec, np.eye(len(w)), atol=1e-10)


@need_ref
def test_plugin_linalg_device_reconstruction(problem):
    """tsvd_family / spectrum with the device algebra installed give the
    host's reconstructions and eigenvalues."""
    from paper_2409_03686_b200 import plugin

    ref = _ref()
    from exitmeasure.estimator import EstimatorBundle, MeasurementSet
    from exitmeasure.geometry import BoundaryPointSet
    from exitmeasure.tsvd import spectrum, tsvd_family
    from exitmeasure.weights import WeightFamily

    a1, sigma1, nu = problem
    rng = np.random.default_rng(7)
    mp, m1 = a1.shape
    pts = rng.normal(size=(mp, 2))
    meas = MeasurementSet(pts, rng.normal(size=mp), nu, np.zeros((0, 2)), np.zeros(0))
    fam1 = WeightFamily("voronoi", BoundaryPointSet(rng.normal(size=(m1, 2)), np.zeros(m1),
                                                    np.zeros(m1)), sigma1)
    z = np.zeros(mp)

    def bundle():
        return EstimatorBundle(a1, np.zeros((mp, 0)), sigma1, ref.estimator._gram(a1, sigma1, nu),
                               nu, 10_000, 1e-5, 0, z, z, z)

    saved = (ref.estimator._gram, ref.tsvd.svd, ref.tsvd.sym_eig, ref.linalg.svd)
    hb = bundle()
    host_fam = tsvd_family(hb, meas, fam1, [3, 8, 20])
    host_sp = spectrum(hb)
    try:
        plugin.install_linalg()
        b = bundle()  # Gram from the device now
        assert np.max(np.abs(b.lambda_nu - hb.lambda_nu)) <= 1e-12 * np.max(np.abs(hb.lambda_nu))
        dev_fam = tsvd_family(b, meas, fam1, [3, 8, 20])
        dev_sp = spectrum(b)
    finally:
        (ref.estimator._gram, ref.tsvd.svd, ref.tsvd.sym_eig, ref.linalg.svd) = saved
    scale = np.max(np.abs(host_fam.solutions))
    assert np.max(np.abs(dev_fam.solutions - host_fam.solutions)) <= 1e-8 * scale
    assert dev_fam.rank == host_fam.rank
    assert np.allclose(dev_sp.eigenvalues, host_sp.eigenvalues, rtol=1e-10,
                       atol=1e-13 * host_sp.eigenvalues[0])
