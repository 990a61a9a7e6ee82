"""High-power parity of the production FP32 tangent / rolling chains
(formerly tools/diag/soak_tangent.py, now in the suite): per config, 1e7 GPU walks
per pole against 2e5 .. 2e6 walks per pole of the C oracle (the reference's
FP64 walk-on-ellipsoids chain, S/_kernel.pyx:163-197, brute-force Voronoi
binning, all host threads).  Two statistics per config: the per-pole
Gamma_1 hit fractions (two-sample z, Bonferroni over the poles) and per-pole
two-sample chi^2 over 64 groups of consecutive bins (Fisher-combined).
Family-wise level 1e-4 per statistic (fixed seeds: deterministic per build)."""

import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

RUNS = [(2, 16, 2_000_000), (3, 16, 1_000_000), (4, 16, 500_000), (5, 8, 200_000)]
N_GPU = 10_000_000
LEVEL = 1e-4


def _generic(sd, d):
    if sd.size == 0:
        return (np.zeros((0, d)), np.array([[0, 0, 0]]), np.zeros((1, 4)))
    return (sd.anchors, np.array([[0, 0, sd.size]]), np.zeros((1, 4)))


@pytest.mark.parametrize("idx,n_poles,n_ref", RUNS)
def test_tangent_chain_soak(oracle, idx, n_poles, n_ref):
    from scipy import stats

    from paper_2409_03686_b200 import _native, backend as B, configs

    _native.require_device(0)
    cfg = configs.get(idx).subset(n_poles)
    geom = B.pack_geometry(cfg.dom)
    s0, s1 = B.pack_side(cfg.fam0, cfg.d, cfg.eps), B.pack_side(cfg.fam1, cfg.d, cfg.eps)
    with B.Plan(geom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, 10**6, s0, s1,
                precision="fp32") as plan:
        assert plan.chain == "tangent"
        g = plan.run(cfg.seed + 1000, N_GPU).counts.astype(np.float64)
    o0, o1, *_r, oerr = oracle.run_accumulate_packed(
        geom.gi, geom.gf, geom.comp_side, cfg.kt.k_sqrt, cfg.poles, cfg.seed, cfg.eps, 10**6,
        n_ref, _generic(s0, cfg.d), _generic(s1, cfg.d), threads=os.cpu_count() or 1)
    assert oerr is None
    r = np.concatenate([o0, o1], axis=1).astype(np.float64)
    assert (g.sum(1) == N_GPU).all() and (r.sum(1) == n_ref).all()
    n0 = s0.size
    fg = cfg.split(g[:, :n0], g[:, n0:])[1].sum(1) / N_GPU
    fr = cfg.split(r[:, :n0], r[:, n0:])[1].sum(1) / n_ref
    p = (fg * N_GPU + fr * n_ref) / (N_GPU + n_ref)
    z = (fg - fr) / np.sqrt(p * (1 - p) * (1 / N_GPU + 1 / n_ref))
    assert np.abs(z).max() <= stats.norm.isf(LEVEL / (2 * n_poles)), z
    edges = np.linspace(0, g.shape[1], 65).astype(int)[:-1]
    gg, gr = np.add.reduceat(g, edges, axis=1), np.add.reduceat(r, edges, axis=1)
    pv = np.array([stats.chi2_contingency(np.vstack([gg[i], gr[i]])[:, (gg[i] + gr[i]) > 0])[1]
                   for i in range(n_poles)])
    assert pv.min() > LEVEL / n_poles, pv
    assert stats.combine_pvalues(pv)[1] > LEVEL, pv
