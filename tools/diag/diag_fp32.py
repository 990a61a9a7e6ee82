"""Diagnostic: dump FP32 count rows for reduced configs (GPU box) so the
statistical comparison against the oracle can be studied off-box."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2409_03686_b200 import backend as B, configs  # noqa: E402

out = {}
for idx, n_poles, n in [(2, 32, 10**6), (3, 32, 10**6), (4, 16, 400_000), (5, 8, 200_000)]:
    cfg = configs.get(idx).subset(n_poles)
    s0 = B.pack_side(cfg.fam0, cfg.d, cfg.eps)
    s1 = B.pack_side(cfg.fam1, cfg.d, cfg.eps)
    for chain in ("woe", "max"):
        r = B.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.seed, cfg.eps, 10**6, n,
                             s0, s1, precision="fp32", chain=chain)
        out[f"cfg{idx}.{chain}"] = r.counts
        out[f"cfg{idx}.{chain}.steps"] = r.steps_sum
        print(idx, chain, r.steps_sum.sum() / (n * cfg.n_poles), r.kernel_ms, flush=True)
    x, st, comp = B.run_exits(cfg.dom, cfg.kt.k_sqrt, cfg.poles[0], 0, cfg.seed, cfg.eps, 10**6,
                              20000, precision="fp32", chain="woe")
    out[f"cfg{idx}.exits"] = x
np.savez_compressed(sys.argv[1], **out)
