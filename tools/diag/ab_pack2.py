"""A/B of the packed two-walks-per-lane kernel against the one-walk-per-lane
kernel on cfg3: counts equal bit for bit?  kernel times."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2409_03686_b200 import _native, backend, configs

def run(cfgno, n_rep, flags, reps=3):
    cfg = configs.get(cfgno)
    geom = backend.pack_geometry(cfg.dom)
    s0 = backend.pack_side(cfg.fam0, cfg.d, cfg.eps)
    s1 = backend.pack_side(cfg.fam1, cfg.d, cfg.eps)
    plan = backend.Plan(geom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, 10**6, s0, s1,
                        precision="fp32", chain="tangent", device=0, flags=flags)
    row = plan.n0 + plan.n1
    counts = torch.zeros((cfg.n_poles, row), dtype=torch.int64, device="cuda")
    stats = torch.zeros((3, cfg.n_poles), dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        plan.run_device(cfg.seed, n_rep, counts.data_ptr(), stats.data_ptr(), st.cuda_stream, 0)
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return counts.cpu().numpy(), stats.cpu().numpy(), min(ts), cfg.n_poles * n_rep

for cfgno, n_rep in ((3, 20000), (3, 1000000)):
    c2, s2, t2, n = run(cfgno, n_rep, 0)
    c1, s1, t1, _ = run(cfgno, n_rep, _native.EM_FLAG_ONE_WALK_PER_LANE)
    print(f"cfg{cfgno} n_rep={n_rep}: packed {t2:.3f} ms ({n / t2 / 1e6:.2f}e9 walks/s)  one-lane {t1:.3f} ms "
          f"({n / t1 / 1e6:.2f}e9 walks/s)  speedup {t1 / t2:.3f}", flush=True)
    print("  rows sum ok:", bool((c2.sum(1) == n_rep).all()), bool((c1.sum(1) == n_rep).all()),
          " counts equal:", bool((c1 == c2).all()), " max |diff|:", int(np.abs(c1 - c2).max()),
          " stats equal:", bool((s1 == s2).all()),
          " steps/walk:", s2[0].sum() / n, s1[0].sum() / n, flush=True)
