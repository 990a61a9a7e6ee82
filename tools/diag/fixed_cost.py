"""Fixed cost of one run (launch, ramp-up, tail): kernel-region time of the
cfg's full pole set at several walk counts per pole, least-squares T = a + b n.
python tools/fixed_cost.py [cfg]   (GPU box)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2409_03686_b200 import backend as B, configs  # noqa: E402

cfg = configs.get(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
geom = B.pack_geometry(cfg.dom)
s0 = B.pack_side(cfg.fam0, cfg.d, cfg.eps)
s1 = B.pack_side(cfg.fam1, cfg.d, cfg.eps)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream()
plan = B.Plan(geom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, 10**6, s0, s1, precision="fp32")
counts = torch.zeros((cfg.n_poles, plan.n0 + plan.n1), dtype=torch.int64, device="cuda")
stats = torch.zeros((3, cfg.n_poles), dtype=torch.int64, device="cuda")
ns, ts = [], []
for n in (1, 100, 1000, 3000, 10000, 30000, 100000):
    ms = []
    for i in range(13):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        plan.run_device(cfg.seed, n, counts.data_ptr(), stats.data_ptr(), stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        if i >= 3:
            ms.append(a.elapsed_time(b))
    t = float(np.median(ms))
    print(f"{cfg.name}: {cfg.n_poles} poles x {n}: {t * 1e3:.1f} us")
    if n >= 1000:
        ns.append(n * cfg.n_poles)
        ts.append(t)
b, a = np.polyfit(ns, ts, 1)
print(f"fit over n >= 1000: fixed {a * 1e3:.1f} us + {b * 1e9:.3f} ns/walk")
