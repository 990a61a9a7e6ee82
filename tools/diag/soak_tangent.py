"""Parity soak of the FP32 tangent chains against the C oracle (the reference's
FP64 walk-on-ellipsoids chain, brute-force Voronoi binning) at large walk
counts, cfg2..cfg5 (GPU box; the oracle runs on all host threads):
per-pole Gamma_1 hit fractions (z-scores) and two-sample chi^2 over 64 groups
of consecutive bins per pole.   python tools/soak_tangent.py [scale]"""
import dataclasses
import os
import sys
import time
from pathlib import Path

import numpy as np
from scipy import stats

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402  (test infrastructure: the checker)
from paper_2409_03686_b200 import backend as B, configs  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
only = [int(c) for c in sys.argv[2].split(",")] if len(sys.argv) > 2 else None
chains = sys.argv[3].split(",") if len(sys.argv) > 3 else [None]
RUNS = [(2, 16, 2_000_000), (3, 16, 1_000_000), (4, 16, 500_000), (5, 8, 200_000)]
N_GPU = int(10_000_000 * max(scale, 1.0))
SEED = int(os.environ.get("SOAK_SEED", "0"))  # offset of both runs' seeds


def generic(sd, d):
    if sd.size == 0:
        return (np.zeros((0, d)), np.array([[0, 0, 0]]), np.zeros((1, 4)))
    return (sd.anchors, np.array([[0, 0, sd.size]]), np.zeros((1, 4)))


for idx, n_poles, n_ref in RUNS:
    if only and idx not in only:
        continue
    n_ref = int(n_ref * scale)
    ref_cache = None
    for ch in chains:
        cfg = configs.get(idx).subset(n_poles)
        if os.environ.get("SOAK_EPS"):  # eps study: the chains' O(eps) shell effects
            cfg = dataclasses.replace(cfg, eps=float(os.environ["SOAK_EPS"]))
        geom = B.pack_geometry(cfg.dom)
        s0, s1 = B.pack_side(cfg.fam0, cfg.d, cfg.eps), B.pack_side(cfg.fam1, cfg.d, cfg.eps)
        with B.Plan(geom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, 10**6, s0, s1, precision="fp32",
                    chain=ch) as plan:
            chain = plan.chain
            g = plan.run(cfg.seed + 1000 + SEED, N_GPU).counts.astype(np.float64)
        t = time.time()
        if ref_cache is None:
            ref_cache = O.run_accumulate_packed(
                geom.gi, geom.gf, geom.comp_side, cfg.kt.k_sqrt, cfg.poles, cfg.seed + SEED, cfg.eps,
                10**6, n_ref, generic(s0, cfg.d), generic(s1, cfg.d))
        o0, o1, oss, *_r, oerr = ref_cache
        t_ref = time.time() - t
        assert oerr is None
        r = np.concatenate([o0, o1], axis=1).astype(np.float64)
        assert (g.sum(1) == N_GPU).all() and (r.sum(1) == n_ref).all()
        n0 = s0.size
        fg = cfg.split(g[:, :n0], g[:, n0:])[1].sum(1) / N_GPU
        fr = cfg.split(r[:, :n0], r[:, n0:])[1].sum(1) / n_ref
        p = (fg * N_GPU + fr * n_ref) / (N_GPU + n_ref)
        z = (fg - fr) / np.sqrt(p * (1 - p) * (1 / N_GPU + 1 / n_ref))
        edges = np.linspace(0, g.shape[1], 65).astype(int)[:-1]
        gg, gr = np.add.reduceat(g, edges, axis=1), np.add.reduceat(r, edges, axis=1)
        pv = np.array([stats.chi2_contingency(np.vstack([gg[i], gr[i]])[:, (gg[i] + gr[i]) > 0])[1]
                       for i in range(n_poles)])
        print(f"cfg{idx} {chain}: {n_poles} poles, GPU {N_GPU:.0e} vs oracle {n_ref:.1e} walks/pole "
              f"(oracle {t_ref:.1f} s); Gamma_1 fraction GPU {fg.mean():.5f} oracle {fr.mean():.5f}, "
              f"max |z| {np.abs(z).max():.2f}, sum z^2 p {stats.chi2.sf((z ** 2).sum(), n_poles):.3g}; "
              f"64-group chi^2 p min {pv.min():.3g} median {np.median(pv):.3g} Fisher "
              f"{stats.combine_pvalues(pv)[1]:.3g}", flush=True)
