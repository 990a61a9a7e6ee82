"""Kernel time of the packed and the one-walk-per-lane kernels over job sizes."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2409_03686_b200 import _native, backend, configs

def run(cfgno, n_rep, flags, reps=5):
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
    return min(ts), cfg.n_poles * n_rep

cfgno = int(sys.argv[1])
for n_rep in [int(x) for x in sys.argv[2:]]:
    import os
    xf = int(os.environ.get("XF", "0"))
    t2, n = run(cfgno, n_rep, xf)
    t1, _ = run(cfgno, n_rep, xf | _native.EM_FLAG_ONE_WALK_PER_LANE)
    print(f"cfg{cfgno} n_rep={n_rep}: packed {t2:.4f} ms ({n / t2 / 1e6:.2f}e9/s)  one {t1:.4f} ms ({n / t1 / 1e6:.2f}e9/s)  speedup {t1 / t2:.3f}", flush=True)
