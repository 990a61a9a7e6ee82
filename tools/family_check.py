"""Small launches of every walk-kernel family: cfg1-cfg5 on the FP32
production kernel (default chain and the max chain), the REF64 mirror on
cfg1 / cfg2, the exits kernel and the point binner, each checked for exact
row sums (every walk in exactly one valid bin of its own row), in-domain
exits and in-range bin indices.  compute-sanitizer is closed on the GPU pool,
so these invariants are the out-of-bounds evidence: python tools/family_check.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2409_03686_b200 import _native, backend, configs

_native.require_device(0)
for c in (1, 2, 3, 4, 5):
    cfg = configs.get(c).subset(4, 512)
    geom = backend.pack_geometry(cfg.dom)
    s0 = backend.pack_side(cfg.fam0, cfg.d, cfg.eps)
    s1 = backend.pack_side(cfg.fam1, cfg.d, cfg.eps)
    runs = [("fp32", None), ("fp32", "max")] + ([("ref64", None)] if c <= 2 else [])
    for prec, chain in runs:
        try:
            plan = backend.Plan(geom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, 10**6, s0, s1,
                                precision=prec, chain=chain)
        except Exception as e:  # a chain a family does not offer
            print(f"cfg{c} {prec}/{chain}: not offered ({e})")
            continue
        with plan:
            r = plan.run(cfg.seed, cfg.n_rep)
            assert np.array_equal(r.counts.sum(1), np.full(cfg.n_poles, cfg.n_rep)), (c, prec)
            x, steps, comp = plan.exits(cfg.seed, 64)
            assert len(steps) == cfg.n_poles * 64
            assert np.all(steps >= 0) and np.all(np.isfinite(x)), (c, prec)
            comp_b, side_b, bin_b = plan.bin_points(x[: min(len(x), 256)])
            nb = np.where(side_b == 0, plan.n0, plan.n1)
            assert np.all((bin_b >= 0) & (bin_b < nb)), (c, prec)
            print(f"cfg{c} {prec}/{plan.chain}: rows exact, exits {x.shape}, binned {len(bin_b)} in range")
# the packed two-walks-per-lane kernels (cfg2 box, cfg3 annulus, a disc without
# hole), both schedulers, forced at this small size; equal to the one-walk kernel
from paper_2409_03686_b200.geometry import Ball, Domain, circle_points

cases = []
for c in (2, 3):
    cfg = configs.get(c).subset(6, 3000)
    cases.append((f"cfg{c}", cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, cfg.fam0, cfg.fam1, cfg.d,
                  cfg.seed, cfg.n_rep))
cfg = configs.get(3)
cases.append(("disc", Domain(2, Ball(np.zeros(2), 1.0), (), frozenset()), cfg.kt.k_sqrt,
              0.8 * cfg.poles[:6], cfg.eps, None,
              circle_points(np.zeros(2), 1.0, 1024, component=0, phase=0.5), 2, cfg.seed, 5000))
for name, dom, ks, poles, eps, f0, f1, d, seed, n_rep in cases:
    geom = backend.pack_geometry(dom)
    s0 = backend.pack_side(f0, d, eps)
    s1 = backend.pack_side(f1, d, eps)
    for sched in (_native.EM_FLAG_PERSISTENT, _native.EM_FLAG_POLE_BLOCKS):
        res = []
        for lanes in (_native.EM_FLAG_TWO_WALKS_PER_LANE, _native.EM_FLAG_ONE_WALK_PER_LANE):
            with backend.Plan(geom, ks, poles, eps, 10**6, s0, s1, precision="fp32",
                              flags=sched | lanes) as plan:
                r = plan.run(seed, n_rep)
                res.append((r, plan.last_walks_per_lane(), plan.last_scheduler()))
        assert res[0][1] == 2 and res[1][1] == 1, name
        assert np.array_equal(res[0][0].counts.sum(1), np.full(len(poles), n_rep)), name
        assert np.array_equal(res[0][0].counts, res[1][0].counts), name
        assert np.array_equal(res[0][0].steps_sum, res[1][0].steps_sum), name
        print(f"{name} packed ({res[0][2]}): rows exact, equal to the one-walk kernel")
print("family_check ok")
