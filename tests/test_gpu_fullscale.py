"""Entry-wise parity at BASELINE scale, and the spectral criterion on the
production chain (north_star: "each entry of A agrees with the reference's
estimate within 4 binomial standard errors"; "the leading singular values
and the reconstructed u1 agree within a stated relative tolerance").

* cfg2 at its FULL size (256 poles x 1e5 walks, 512 bins) on the FP32
  tangent chain against one full run of the reference itself (oracle/_ref:
  the unmodified exitmeasure package, its compiled Cython kernel, all host
  threads -- T/test_backend.py:78-86's comparison at BASELINE scale).
* cfg3 and cfg4 (64 poles x 1e6 GPU walks) against 1e5 reference walks per
  pole; cfg5 (64 poles x 1e6) against 1e5 walks per pole of the C oracle
  (no reference expression exists for the L-box).
* SURVEY Appendix B's three statistics on every comparison: the number of
  entries beyond |z| = 4 against the binomial 99.9% quantile of a perfect
  implementation, per-row chi^2 homogeneity p-values (KS-uniform), and the
  extreme entry against the Bonferroni level.  Entry-wise tails use the
  EXACT conditional binomial test (p-values, then z-equivalents): the normal
  z is wrong at the low counts of far-side bins.
* cfg2, tangent chain: sigma_1..sigma_8 of A over 8 GPU seeds against 6
  full-scale reference seeds (pooled two-sample t-test per singular value,
  Bonferroni over the 8), and the u1 reconstruction (the reference's own
  tsvd_family, S/tsvd.py:93-130, r = 3, 4, 5) of a K-harmonic u likewise.

Summaries go to gpurun_out/fullscale_*.json (profiles/ keeps the round's).
"""

import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import pytest

from helpers import exact_two_sample_p, exceed_quantile, row_chi2_pvalues

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref"
THREADS = os.cpu_count() or 1
P_Z4 = 6.334248366623996e-05


@pytest.fixture(scope="module")
def B():
    from paper_2409_03686_b200 import _native, backend

    _native.require_device(0)
    return backend


def _ref_module():
    if not (REF / "exitmeasure").exists():
        pytest.skip("oracle/_ref not built")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import exitmeasure.backend as rb

    assert rb.BACKEND == "compiled" and not hasattr(rb, "_em_b200_original")
    return rb


def reference_counts(cfg, n, seed, oracle=None, with_stats=False):
    """(n_poles, n0 + n1) exit counts in this package's column order from the
    reference's own run_accumulate (cfg1-cfg4, SURVEY Appendix A
    expressions) or, for cfg5, from the C oracle (brute-force binning)."""
    from paper_2409_03686_b200 import backend as B

    if cfg.index == 5:
        geom = B.pack_geometry(cfg.dom)
        s0 = B.pack_side(cfg.fam0, 3, cfg.eps)
        s1 = B.pack_side(cfg.fam1, 3, cfg.eps)
        raw0, raw1, *_rest, err = oracle.run_accumulate_packed(
            geom.gi, geom.gf, geom.comp_side, cfg.kt.k_sqrt, cfg.poles, seed, cfg.eps, 10**6, n,
            (s0.anchors, s0.blk, s0.blkf), (s1.anchors, s1.blk, s1.blkf), threads=THREADS)
        assert err is None
        return np.concatenate([raw0, raw1], 1).astype(np.int64)
    rb = _ref_module()
    from exitmeasure.geometry import Ball, Box, BoundaryPointSet, catalog, make_domain, side_points

    if cfg.index == 3:
        dom = catalog("annulus")
        f0 = side_points(dom, "gamma0", [512])
        f1 = side_points(dom, "gamma1", [512])
        assert np.allclose(f0.points, cfg.fam0.points, atol=1e-15)
        assert np.allclose(f1.points, cfg.fam1.points, atol=1e-15)
        s0 = rb.pack_side(f0, 2, cfg.eps)
        s1 = rb.pack_side(f1, 2, cfg.eps)
    else:
        outer = Box(np.array([0.5, 0.5]), 0.5) if cfg.index == 2 else Ball(np.zeros(cfg.d), 1.0)
        dom = make_domain(outer, gamma0=())
        pts = np.ascontiguousarray(cfg.fam1.points)
        s1 = rb.pack_side(BoundaryPointSet(pts, np.zeros(len(pts), int),
                                           np.arange(len(pts), dtype=float), ()), cfg.d, cfg.eps)
        s0 = rb.pack_side(None, cfg.d, cfg.eps)
    r = rb.run_accumulate(dom, cfg.kt.k_sqrt, cfg.poles, seed, cfg.eps, 10**6, n, s0, s1,
                          threads=THREADS)
    counts = np.concatenate([r.raw0, r.raw1], 1).astype(np.int64)
    if with_stats:
        return counts, (r.steps_sum, r.steps_sq_sum, r.steps_max)
    return counts


def appendix_b(gpu, n_gpu, ref, n_ref, label):
    """Appendix B two-sample statistics; returns the summary dict."""
    from scipy import stats

    p = exact_two_sample_p(gpu, n_gpu, ref, n_ref)
    m = p.size
    z_eq = stats.norm.isf(np.clip(p, 1e-300, 1.0) / 2.0)  # |z| with the same tail mass
    rows = row_chi2_pvalues(gpu, n_gpu, ref, n_ref)
    summary = {
        "label": label, "entries": int(m), "n_gpu": int(n_gpu), "n_ref": int(n_ref),
        "exceed_z4": int((p < P_Z4).sum()), "exceed_z4_q999": exceed_quantile(m),
        "max_abs_z_equiv": float(z_eq.max()),
        "bonferroni_z": float(stats.norm.isf(0.025 / m)),
        "min_p": float(p.min()), "bonferroni_p": 0.05 / m,
        "row_chi2_min_p": float(rows.min()), "row_chi2_ks_uniform_p":
            float(stats.kstest(rows, "uniform").pvalue),
        "rows": int(len(rows)),
    }
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    (out / f"fullscale_{label}.json").write_text(json.dumps(summary, indent=1))
    return summary


def _check(s):
    assert s["exceed_z4"] <= s["exceed_z4_q999"], s
    assert s["max_abs_z_equiv"] <= s["bonferroni_z"], s
    assert s["row_chi2_min_p"] > 1e-4 / s["rows"], s
    assert s["row_chi2_ks_uniform_p"] > 1e-3, s


def _gpu_counts(B, cfg, n, seed, chain="tangent"):
    s0 = B.pack_side(cfg.fam0, cfg.d, cfg.eps)
    s1 = B.pack_side(cfg.fam1, cfg.d, cfg.eps)
    r = B.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, seed, cfg.eps, 10**6, n, s0, s1,
                         precision="fp32", chain=chain)
    assert np.array_equal(r.counts.sum(1), np.full(cfg.n_poles, n))
    return r.counts


def test_cfg2_full_scale_against_the_reference(B):
    from paper_2409_03686_b200 import configs

    cfg = configs.get(2)
    gpu = _gpu_counts(B, cfg, cfg.n_rep, cfg.seed)
    t0 = time.perf_counter()
    ref = reference_counts(cfg, cfg.n_rep, cfg.seed + 1)
    s = appendix_b(gpu, cfg.n_rep, ref, cfg.n_rep, "cfg2_full")
    s["reference_seconds"] = time.perf_counter() - t0
    _check(s)


@pytest.mark.parametrize("idx", [3, 4, 5])
def test_large_configs_against_the_reference(B, oracle, idx):
    from paper_2409_03686_b200 import configs

    cfg = configs.get(idx).subset(64)
    gpu = _gpu_counts(B, cfg, 10**6, cfg.seed)
    ref = reference_counts(cfg, 10**5, cfg.seed + 1, oracle)
    _check(appendix_b(gpu, 10**6, ref, 10**5, f"cfg{idx}_64x1e6_vs_1e5"))


# ---------------------------------------------------------------------------
# spectral criterion on the production chain (cfg2, tangent balls)


@pytest.fixture(scope="module")
def cfg2_estimates(B):
    from paper_2409_03686_b200 import configs

    cfg = configs.get(2)
    gpu = [_gpu_counts(B, cfg, cfg.n_rep, 7000 + k) / cfg.n_rep for k in range(8)]
    ref = [reference_counts(cfg, cfg.n_rep, 9000 + k) / cfg.n_rep for k in range(6)]
    return cfg, gpu, ref


def _two_sample_t(g, r):
    """Pooled two-sample t statistic per column and its degrees of freedom."""
    g, r = np.asarray(g), np.asarray(r)
    ng, nr = len(g), len(r)
    sp2 = ((ng - 1) * g.var(0, ddof=1) + (nr - 1) * r.var(0, ddof=1)) / (ng + nr - 2)
    t = (g.mean(0) - r.mean(0)) / np.sqrt(sp2 * (1.0 / ng + 1.0 / nr))
    return t, ng + nr - 2


def test_cfg2_leading_singular_values(cfg2_estimates):
    """sigma_1..8 of the full 256 x 512 A: GPU (8 seeds) and reference (6
    seeds) means agree by a pooled t-test at family-wise level 1e-3, and the
    two seed spreads agree within a factor 3 (the relative spread itself is
    ~1e-4 .. 5e-4)."""
    from scipy import stats

    cfg, gpu, ref = cfg2_estimates
    sv = lambda a: np.linalg.svd(a, compute_uv=False)[:8]  # noqa: E731
    sg = np.array([sv(a) for a in gpu])
    sr = np.array([sv(a) for a in ref])
    t, dof = _two_sample_t(sg, sr)
    crit = stats.t.isf(1e-3 / 16, dof)
    rel = np.abs(sg.mean(0) - sr.mean(0)) / sr.mean(0)
    summary = {"sigma_gpu_mean": sg.mean(0).tolist(), "sigma_ref_mean": sr.mean(0).tolist(),
               "rel_diff": rel.tolist(), "gpu_rel_spread": (sg.std(0, ddof=1) / sg.mean(0)).tolist(),
               "ref_rel_spread": (sr.std(0, ddof=1) / sr.mean(0)).tolist(), "t": t.tolist(),
               "t_crit": float(crit)}
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "fullscale_cfg2_sigma.json").write_text(json.dumps(summary, indent=1))
    (ROOT / "gpurun_out" / "fullscale_cfg2_sigma.json").write_text(json.dumps(summary, indent=1))
    assert np.all(np.abs(t) <= crit), summary
    # equal seed-to-seed variances (two-sided F-test, Bonferroni over the 8)
    f = sg.var(0, ddof=1) / sr.var(0, ddof=1)
    pf = 2 * np.minimum(stats.f.cdf(f, len(sg) - 1, len(sr) - 1),
                        stats.f.sf(f, len(sg) - 1, len(sr) - 1))
    summary["variance_ratio_p"] = pf.tolist()
    (ROOT / "gpurun_out" / "fullscale_cfg2_sigma.json").write_text(json.dumps(summary, indent=1))
    assert np.all(pf > 1e-3 / 8), summary
    assert np.all(rel <= 2e-3), summary


def test_cfg2_reconstructed_u1(cfg2_estimates):
    """u(x) = h(K^{-1/2} x), h(z) = z_1^2 - z_2^2 (K-harmonic): interior data
    at the 256 poles, Dirichlet data on Gamma0 (right, left, bottom edges),
    TSVD reconstruction on Gamma1 (top edge) at r = 3, 4, 5 with the
    reference's own tsvd_family on every A; GPU and reference sigma-weighted
    L2 errors agree by a pooled t-test, and both reconstruct u1."""
    from scipy import stats

    _ref_module()
    from exitmeasure.estimator import EstimatorBundle, _gram, make_measurements
    from exitmeasure.geometry import Box, BoundaryPointSet, make_domain
    from exitmeasure.tsvd import tsvd_family
    from exitmeasure.weights import WeightFamily

    cfg, gpu, ref = cfg2_estimates
    ainv = np.linalg.inv(cfg.kt.k_sqrt)

    def u(p):
        z = p @ ainv.T
        return z[:, 0] ** 2 - z[:, 1] ** 2

    pts = cfg.fam1.points
    c0, c1 = cfg.a0_cols[1], cfg.a1_cols[1]
    g0, g1 = pts[c0], pts[c1]
    sigma1 = cfg.sigma1
    fam1 = WeightFamily("voronoi", BoundaryPointSet(g1, np.zeros(len(g1)),
                                                    np.zeros(len(g1))), sigma1)
    dom = make_domain(Box(np.array([0.5, 0.5]), 0.5), gamma0=())

    def l2rel(a):
        a0, a1 = a[:, c0], a[:, c1]
        meas = make_measurements(dom, cfg.poles, u(cfg.poles), g0, u(g0))
        z = np.zeros(cfg.n_poles)
        b = EstimatorBundle(a1, a0, sigma1, _gram(a1, sigma1, meas.nu), meas.nu, cfg.n_rep,
                            cfg.eps, 0, z, z, z)
        fam = tsvd_family(b, meas, fam1, [3, 4, 5])
        truth = u(g1)
        err = fam.solutions - truth[None, :]
        return np.sqrt((sigma1 * err ** 2).sum(1) / (sigma1 * truth ** 2).sum())

    eg = np.array([l2rel(a) for a in gpu])
    er = np.array([l2rel(a) for a in ref])
    t, dof = _two_sample_t(eg, er)
    crit = stats.t.isf(1e-3 / 6, dof)
    summary = {"l2rel_gpu": eg.tolist(), "l2rel_ref": er.tolist(), "t": t.tolist(),
               "t_crit": float(crit)}
    (ROOT / "gpurun_out" / "fullscale_cfg2_u1.json").write_text(json.dumps(summary, indent=1))
    assert np.all(eg < 0.5) and np.all(er < 0.5), summary
    assert np.all(np.abs(t) <= crit), summary


def test_ref64_reproduces_the_reference_at_full_scale(B):
    """The bit-exact FP64 mirror at BASELINE scale: cfg2 at its full 256 poles
    x 1e5 walks and cfg4 at 64 poles x 1e4, the REFERENCE's own compiled
    kernel (oracle/_ref, all host threads) against this library's REF64 path
    on the same seed -- every count and every step statistic identical."""
    from paper_2409_03686_b200 import configs

    rb = _ref_module()
    for idx, n_poles, n in ((2, None, None), (4, 64, 10_000)):
        cfg = configs.get(idx)
        cfg = cfg.subset(n_poles, n) if n_poles else cfg
        ref, st = reference_counts(cfg, cfg.n_rep, cfg.seed, with_stats=True)
        s0 = B.pack_side(cfg.fam0, cfg.d, cfg.eps)
        s1 = B.pack_side(cfg.fam1, cfg.d, cfg.eps)
        # the reference expression bins by brute force over the generic family
        # (reference_counts): the mirror with the same generic blocks
        g1 = B.SidePack(s1.anchors, np.array([[0, 0, s1.size]], dtype=np.int64),
                        np.zeros((1, 4)), 0, np.zeros(0), 2, np.zeros(1))
        r = B.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.seed, cfg.eps, 10**6,
                             cfg.n_rep, s0, g1, precision="ref64")
        assert np.array_equal(r.counts, ref), idx
        assert np.array_equal(r.steps_sum, st[0]) and np.array_equal(r.steps_sq_sum, st[1])
        assert np.array_equal(r.steps_max, st[2]), idx
