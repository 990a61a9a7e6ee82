"""cfg4 diagnostics: FP32 grid binning vs exact brute force on the same
points, and a large FP32 sample of one pole."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2409_03686_b200 import backend as B, configs  # noqa: E402

cfg = configs.get(4).subset(16)
geom = B.pack_geometry(cfg.dom)
s0 = B.pack_side(cfg.fam0, 3, cfg.eps)
s1 = B.pack_side(cfg.fam1, 3, cfg.eps)
# exits of pole 10 (FP32 walk), binned two ways
x, st, comp = B.run_exits(cfg.dom, cfg.kt.k_sqrt, cfg.poles[10], 10, cfg.seed, cfg.eps, 10**6,
                          200000, precision="fp32")
out = {"x": x}
for prec in ("fp32", "ref64"):
    with B.Plan(geom, cfg.kt.k_sqrt, cfg.poles[:1], cfg.eps, 10**6, s0, s1, precision=prec) as p:
        c, s, b = p.bin_points(x)
    out["bin_" + prec] = b
dis = out["bin_fp32"] != out["bin_ref64"]
print("disagreements fp32-grid vs exact:", int(dis.sum()), "of", len(x))
r = B.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.seed + 7, cfg.eps, 10**6, 2_000_000,
                     s0, s1, precision="fp32", chain="max")
out["counts_max"] = r.counts
r = B.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.seed + 7, cfg.eps, 10**6, 2_000_000,
                     s0, s1, precision="fp32", chain="woe")
out["counts_woe"] = r.counts
np.savez_compressed(sys.argv[1], **out)
print("pole 10 bin 213 rate max/woe:", out["counts_max"][10, 213] / 2e6, out["counts_woe"][10, 213] / 2e6)
