"""Host-side cost of one backend.run_accumulate call (cfg2 geometry, 1 walk
per pole so the kernel is negligible): mean wall time and a cProfile of the
Python layer.  python tools/api_overhead.py  (GPU box)"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2409_03686_b200 import backend as B, configs  # noqa: E402

cfg = configs.get(2)
s0 = B.pack_side(cfg.fam0, cfg.d, cfg.eps)
s1 = B.pack_side(cfg.fam1, cfg.d, cfg.eps)


def call():
    return B.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, cfg.seed, cfg.eps, 10**6, 1, s0, s1,
                            precision="fp32")


for _ in range(50):
    call()
n = 500
t0 = time.perf_counter()
for _ in range(n):
    call()
print(f"run_accumulate, 256 poles x 1 walk: {1e6 * (time.perf_counter() - t0) / n:.1f} us per call")
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    call()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
