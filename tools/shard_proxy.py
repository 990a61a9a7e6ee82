"""Single-GPU proxy of the row-sharded strong-scaling run: rank 0's shard of
an N-GPU run (poles i = 0 mod N, global pole ids) timed alone, L2 flushed
between steps, CUDA events.  Compute-side efficiency T_1 / (N T_N) before the
all-gather.  python tools/shard_proxy.py [cfg] [steps] [rows|reps]   (GPU box)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2409_03686_b200 import backend as B, configs  # noqa: E402

cfg = configs.get(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
geom = B.pack_geometry(cfg.dom)
s0 = B.pack_side(cfg.fam0, cfg.d, cfg.eps)
s1 = B.pack_side(cfg.fam1, cfg.d, cfg.eps)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream()
t1 = None
# "rows": rank 0's cyclic row shard (what a strong-scaled run does);
# "reps": the same walk count as all poles x n_rep / N (contention check:
# the same work spread over every count row)
mode = sys.argv[3] if len(sys.argv) > 3 else "rows"
for n in (1, 2, 4, 8):
    ids = B.np.arange(0, cfg.n_poles, n) if mode == "rows" else B.np.arange(cfg.n_poles)
    n_rep = cfg.n_rep if mode == "rows" else cfg.n_rep // n
    plan = B.Plan(geom, cfg.kt.k_sqrt, cfg.poles[ids], cfg.eps, 10**6, s0, s1, precision="fp32",
                  pole_ids=ids)
    counts = torch.zeros((len(ids), plan.n0 + plan.n1), dtype=torch.int64, device="cuda")
    stats = torch.zeros((3, len(ids)), dtype=torch.int64, device="cuda")
    ms = []
    for i in range(steps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        plan.run_device(cfg.seed, n_rep, counts.data_ptr(), stats.data_ptr(), stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        if i >= 3:
            ms.append(a.elapsed_time(b))
    plan.check()
    t = sorted(ms)[len(ms) // 2]
    t1 = t if n == 1 else t1
    print(f"{cfg.name} {mode} N={n}: {len(ids)} poles x {n_rep}, {t:.4f} ms median, "
          f"compute-side efficiency {t1 / (n * t):.3f}")
    plan.close()
