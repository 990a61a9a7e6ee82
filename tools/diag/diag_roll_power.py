"""High-power check of the rolling-ball chain (cfg4) against the max chain:
python tools/diag_roll_power.py [n_poles] [n_walks]"""
import sys
from pathlib import Path

import numpy as np
from scipy import stats

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2409_03686_b200 import backend as B, configs  # noqa: E402

n_poles = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4_000_000
c = configs.get(4).subset(n_poles)
g = B.pack_geometry(c.dom)
s0, s1 = B.pack_side(c.fam0, 3, c.eps), B.pack_side(c.fam1, 3, c.eps)
res = {}
S = int(sys.argv[3]) if len(sys.argv) > 3 else 7
for chain, seed in (("max", S), ("tangent", S + 1)):
    with B.Plan(g, c.kt.k_sqrt, c.poles, c.eps, 10**6, s0, s1, precision="fp32", chain=chain) as p:
        res[chain] = p.run(seed, n).counts.astype(np.float64)
a, b = res["max"], res["tangent"]
for name, cols in (("Gamma1", slice(1024, 2048)), ("first quarter", slice(0, 512)),
                   ("cols%4==0", slice(0, 2048, 4))):
    fa, fb = a[:, cols].sum(1) / n, b[:, cols].sum(1) / n
    p = (fa + fb) / 2
    z = (fb - fa) / np.sqrt(2 * p * (1 - p) / n)
    print(f"{name}: max {fa.mean():.6f} tangent {fb.mean():.6f}  max|z| {np.abs(z).max():.2f} "
          f"mean z {z.mean():.3f} (sd of mean {1 / np.sqrt(n_poles):.3f}) chi2 p "
          f"{stats.chi2.sf((z ** 2).sum(), n_poles):.3g}")
for groups in (256, 2048):
    edges = np.linspace(0, 2048, groups + 1).astype(int)[:-1]
    ga, gb = np.add.reduceat(a, edges, axis=1), np.add.reduceat(b, edges, axis=1)
    pv = np.array([stats.chi2_contingency(np.vstack([ga[i], gb[i]])[:, (ga[i] + gb[i]) > 0])[1]
                   for i in range(n_poles)])
    print(f"{groups} groups: p min {pv.min():.3g} median {np.median(pv):.3g} fisher "
          f"{stats.combine_pvalues(pv)[1]:.3g}")
