"""Where does the one-shot API call spend its time? (GPU box)"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2409_03686_b200 import backend as B, configs  # noqa: E402

cfg = configs.get(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
for it in range(4):
    t0 = time.perf_counter()
    geom = B.pack_geometry(cfg.dom)
    s0 = B.pack_side(cfg.fam0, cfg.d, cfg.eps)
    s1 = B.pack_side(cfg.fam1, cfg.d, cfg.eps)
    t1 = time.perf_counter()
    plan = B.Plan(geom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, 10**6, s0, s1, precision="fp32")
    t2 = time.perf_counter()
    r = plan.run(cfg.seed, cfg.n_rep)
    t3 = time.perf_counter()
    plan.close()
    t4 = time.perf_counter()
    print(f"iter {it}: pack {1e3*(t1-t0):.2f} ms, plan {1e3*(t2-t1):.2f} ms, run {1e3*(t3-t2):.2f} ms "
          f"(kernel {r.kernel_ms:.2f} ms), close {1e3*(t4-t3):.2f} ms, total {1e3*(t4-t0):.2f} ms")
