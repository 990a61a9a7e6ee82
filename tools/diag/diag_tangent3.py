"""Diagnostic (GPU box): the 3D tangent-ball chain against the max chain
(itself checked against the oracle in the GPU suite) at high walk counts --
steps per walk, kernel time, per-pole Gamma_1 hit fractions and grouped-bin
two-sample chi^2 -- on cfg5 (L-box) and an off-centre anisotropic 3D box.
python tools/diag_tangent3.py [n_walks]"""
import sys
from pathlib import Path

import numpy as np
from scipy import stats

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2409_03686_b200 import backend as B, configs  # noqa: E402
from paper_2409_03686_b200.conductivity import make_tensor  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10**6


def compare(name, dom_args, k, poles, eps, s0, s1, n, n1_cols, groups=64):
    geom = dom_args if isinstance(dom_args, B.GeomPack) else B.pack_geometry(dom_args)
    res = {}
    for chain in ("max", "tangent"):
        with B.Plan(geom, k, poles, eps, 10**6, s0, s1, precision="fp32", chain=chain) as plan:
            assert plan.chain == chain, (plan.chain, chain)
            plan.run(11, n)
            r = plan.run(12 if chain == "max" else 13, n)
        res[chain] = r
        print(f"{name} {chain}: steps/walk {r.steps_sum.sum() / (n * len(poles)):.3f} "
              f"kernel {r.kernel_ms:.3f} ms  walks/s {n * len(poles) / r.kernel_ms * 1e3:.3e}",
              flush=True)
    a, b = res["max"].counts.astype(np.float64), res["tangent"].counts.astype(np.float64)
    assert (a.sum(1) == n).all() and (b.sum(1) == n).all()
    # Gamma_1 fraction per pole
    f1a, f1b = a[:, -n1_cols:].sum(1) / n, b[:, -n1_cols:].sum(1) / n
    p = (f1a + f1b) / 2
    z = (f1b - f1a) / np.sqrt(np.maximum(2 * p * (1 - p) / n, 1e-300))
    print(f"{name}: Gamma1 fraction max {f1a.mean():.5f} tangent {f1b.mean():.5f}; "
          f"z per pole max |z| {np.abs(z).max():.2f}, mean z {z.mean():.2f}")
    # grouped bins: contiguous index ranges
    cols = a.shape[1]
    edges = np.linspace(0, cols, groups + 1).astype(int)
    ga = np.add.reduceat(a, edges[:-1], axis=1)
    gb = np.add.reduceat(b, edges[:-1], axis=1)
    pv = []
    for i in range(a.shape[0]):
        tab = np.vstack([ga[i], gb[i]])
        keep = tab.sum(0) > 0
        chi2, pval, _, _ = stats.chi2_contingency(tab[:, keep])
        pv.append(pval)
    pv = np.array(pv)
    print(f"{name}: grouped chi^2 ({groups} groups) p-values min {pv.min():.3g} "
          f"median {np.median(pv):.3g}; fisher combined p "
          f"{stats.combine_pvalues(pv)[1]:.3g}", flush=True)
    return res


# cfg5 (L-box)
cfg = configs.get(5).subset(16)
s0 = B.pack_side(cfg.fam0, 3, cfg.eps)
s1 = B.pack_side(cfg.fam1, 3, cfg.eps)
compare("cfg5", cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, s0, s1, n, len(cfg.fam1))

# cfg3 (annulus: rolling disks, disks tangent to the hole)
c3 = configs.get(3).subset(16)
compare("cfg3", c3.dom, c3.kt.k_sqrt, c3.poles, c3.eps, B.pack_side(c3.fam0, 2, c3.eps),
        B.pack_side(c3.fam1, 2, c3.eps), n, 512)

# cfg4 (ball, rolling balls)
c4 = configs.get(4).subset(16)
compare("cfg4", c4.dom, c4.kt.k_sqrt, c4.poles, c4.eps, B.pack_side(c4.fam0, 3, c4.eps),
        B.pack_side(c4.fam1, 3, c4.eps), n, 1024)

# off-centre anisotropic 3D box with generic anchors
rng = np.random.default_rng(5)
c, h = np.array([0.3, -0.2, 0.1]), 0.4
pts = c + rng.uniform(-h, h, size=(600, 3))
ax = np.arange(600) % 3
pts[np.arange(600), ax] = c[ax] + np.where(rng.random(600) < 0.5, -h, h)
blk = np.array([[0, 0, 600]], dtype=np.int64)
side0 = B.SidePack(pts, blk, np.zeros((1, 4)), 0, np.zeros(0), 2)
side1 = B.SidePack(np.zeros((0, 3)), np.array([[0, 0, 0]], dtype=np.int64), np.zeros((1, 4)), 0,
                   np.zeros(0), 2)
k = make_tensor(np.array([[4.0, -1.5, 0.8], [-1.5, 1.0, -0.3], [0.8, -0.3, 0.6]])).k_sqrt
gi = np.array([3, 1, 0], dtype=np.int64)
gf = np.concatenate([c, [h]])
geom = B.GeomPack(gi, gf, np.array([0], dtype=np.int8))
poles = c + rng.uniform(-0.3, 0.3, size=(8, 3))
compare("box3d", geom, k, poles, 1e-5, side0, side1, n, 300, groups=60)

# exits of the tangent chain stay in the eps-shell of the closure
x, st, comp = B.run_exits(cfg.dom, cfg.kt.k_sqrt, cfg.poles[0], 0, cfg.seed, cfg.eps, 10**6,
                          200_000, precision="fp32", chain="tangent")
d_box = np.minimum(x, 1.0 - x).min(1)
notch = np.sqrt(np.maximum(0.5 - x[:, 0], 0) ** 2 + np.maximum(0.5 - x[:, 1], 0) ** 2)
inside_notch = (x[:, 0] > 0.5) & (x[:, 1] > 0.5)
dist = np.minimum(d_box, np.where(inside_notch, -np.minimum(x[:, 0] - 0.5, x[:, 1] - 0.5), notch))
print(f"cfg5 exits: max boundary distance {dist.max():.3g} (eps {cfg.eps:g}), "
      f"min {dist.min():.3g}, mean steps {st.mean():.2f}")
