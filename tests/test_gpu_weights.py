"""Cell measures sigma by GPU-binned boundary quadrature (SURVEY §8f item
2): exact where the cells are known in closed form, consistent between the
exact REF64 rule and the FP32 binner, and defined for the unstructured
families the reference rejects (cfg4 Fibonacci cells, cfg5 squares)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def W():
    from paper_2409_03686_b200 import _native, weights

    _native.require_device(0)
    return weights


@pytest.mark.parametrize("idx", [1, 2, 3])
def test_sigma_closed_form_2d(W, idx):
    from paper_2409_03686_b200 import configs

    cfg = configs.get(idx)
    s0, s1 = W.cell_measures(cfg.dom, cfg.fam0, cfg.fam1, cfg.eps)
    a0, a1 = cfg.split(s0[None, :], s1[None, :])
    assert np.allclose(a1[0], cfg.sigma1, rtol=2e-2)
    assert abs((s0.sum() + s1.sum()) - {1: 2 * np.pi, 2: 4.0, 3: 3 * np.pi}[idx]) < 1e-9


def test_sigma_lbox_squares_exact(W):
    """cfg5: every notch-face cell is a 1/64 square (1/4096), every outer
    cell a 1/30 square (1/900): side-first binning never crosses faces."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(5)
    # a 1/960 midpoint grid nests in both the 1/30 and the 1/64 squares
    s0, s1 = W.cell_measures(cfg.dom, cfg.fam0, cfg.fam1, cfg.eps, spacing=1.0 / 960)
    assert np.allclose(s1, 1.0 / 4096, rtol=1e-9, atol=0)
    assert np.allclose(s0, 1.0 / 900, rtol=1e-9, atol=0)


def test_sigma_fibonacci_hemispheres(W):
    """cfg4: each hemisphere carries 2 pi; interior Fibonacci cells are
    close to equal-area (equatorial rings deviate);
    REF64 and FP32 binning agree."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(4)
    s0, s1 = W.cell_measures(cfg.dom, cfg.fam0, cfg.fam1, cfg.eps, samples_per_anchor=200)
    up, lo = s1[:1024], s1[1024:]
    assert abs(up.sum() - 2 * np.pi) < 2e-3 and abs(lo.sum() - 2 * np.pi) < 2e-3
    mean = 2 * np.pi / 1024
    z = cfg.fam1.points[:1024, 2]
    band = (z > 0.2) & (z < 0.9)  # away from the equator rings and the (under-resolved) cap
    assert np.median(np.abs(up / mean - 1)) < 0.05
    assert np.abs(up[band] / mean - 1).max() < 0.25
    f0, f1 = W.cell_measures(cfg.dom, cfg.fam0, cfg.fam1, cfg.eps, samples_per_anchor=200,
                             precision="fp32")
    assert np.allclose(f1, s1, rtol=2e-2, atol=2e-5)
