"""Find a (pole, replicate) whose walk differs between the packed and the
one-walk-per-lane kernels (bisection on the replicate range)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2409_03686_b200 import _native, backend, configs

cfg = configs.get(3)
geom = backend.pack_geometry(cfg.dom)
s0 = backend.pack_side(cfg.fam0, cfg.d, cfg.eps)
s1 = backend.pack_side(cfg.fam1, cfg.d, cfg.eps)

def mk(flags, ids):
    return backend.Plan(geom, cfg.kt.k_sqrt, cfg.poles[ids], cfg.eps, 10**6, s0, s1,
                        precision="fp32", chain="tangent", device=0, flags=flags, pole_ids=ids)

def run(plan, start, n):
    row = plan.n0 + plan.n1
    counts = torch.zeros((plan.n_poles, row), dtype=torch.int64, device="cuda")
    stats = torch.zeros((3, plan.n_poles), dtype=torch.int64, device="cuda")
    plan.run_device(cfg.seed, n, counts.data_ptr(), stats.data_ptr(), torch.cuda.current_stream().cuda_stream, start)
    torch.cuda.synchronize()
    return counts.cpu().numpy(), stats.cpu().numpy()

ids = np.arange(cfg.n_poles)
p2, p1 = mk(0, ids), mk(_native.EM_FLAG_ONE_WALK_PER_LANE, ids)
n = 20000
c2, t2 = run(p2, 0, n)
c1, t1 = run(p1, 0, n)
bad = np.nonzero((c1 != c2).any(1) | (t1 != t2).any(0))[0]
print("poles that differ:", bad[:20], len(bad))
for pole in bad[:3]:
    ids1 = np.array([pole])
    q2, q1 = mk(0, ids1), mk(_native.EM_FLAG_ONE_WALK_PER_LANE, ids1)
    lo, hi = 0, n
    while hi - lo > 1:
        mid = (lo + hi) // 2
        a2, b2 = run(q2, lo, mid - lo)
        a1, b1 = run(q1, lo, mid - lo)
        if (a1 != a2).any() or (b1 != b2).any():
            hi = mid
        else:
            lo = mid
    a2, b2 = run(q2, lo, 1)
    a1, b1 = run(q1, lo, 1)
    print(f"pole {pole} replicate {lo}: packed bin {np.nonzero(a2[0])[0]} steps {b2[0, 0]}; one-lane bin {np.nonzero(a1[0])[0]} steps {b1[0, 0]}")
    ex = backend.run_exits if hasattr(backend, "run_exits") else None
    try:
        r = q1.exits(cfg.seed, 1, rep_start=lo)
        print("  one-lane exit:", r)
    except Exception as e:
        print("  exits:", repr(e)[:200])
