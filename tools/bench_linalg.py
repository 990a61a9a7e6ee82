"""Host (reference, numpy/LAPACK) vs device (spectral.py) Gram / SVD / eigh at
a BASELINE size: python tools/bench_linalg.py [M] [M1]  (GPU box)."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
from paper_2409_03686_b200 import spectral  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
m1 = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
rng = np.random.default_rng(1)
a1 = rng.binomial(10**6, rng.dirichlet(np.full(m1, 0.3), size=m) * 0.7) / 1e6
sigma1 = rng.uniform(0.5, 1.5, m1) / m1
nu = np.full(m, 1 / np.sqrt(m))
out = {"M": m, "M1": m1, "host_threads": os.cpu_count()}
try:
    from exitmeasure import estimator, linalg
except Exception as e:  # pragma: no cover
    estimator = linalg = None
    out["host"] = f"reference unavailable: {e}"


def timed(f, reps=3):
    f()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = f()
        t.append(time.perf_counter() - t0)
    return min(t), r


import torch  # noqa: E402

def dev_sync(f):
    def g():
        r = f()
        torch.cuda.synchronize()
        return r
    return g


out["device_gram_s"], g_dev = timed(dev_sync(lambda: spectral.gram(a1, sigma1, nu)))
out["device_gram_resident_s"], _ = timed(dev_sync(lambda: spectral.gram_device(
    torch.as_tensor(a1, device="cuda"), sigma1, nu)))
mm = (nu[:, None] * a1) / np.sqrt(sigma1)[None, :]
out["device_svd_s"], (u, s, v) = timed(dev_sync(lambda: spectral.svd(mm)), reps=1)
out["device_eigh_s"], (w, _) = timed(dev_sync(lambda: spectral.sym_eig(g_dev)), reps=1)
if estimator is not None:
    out["host_gram_s"], g_host = timed(lambda: estimator._gram(a1, sigma1, nu), reps=1)
    out["host_svd_s"], (_, s_h, _) = timed(lambda: linalg.svd(mm), reps=0 or 1)
    out["host_eigh_s"], e_h = timed(lambda: linalg.sym_eig(g_host), reps=1)
    out["gram_max_rel_diff"] = float(np.max(np.abs(g_dev - g_host)) / np.max(np.abs(g_host)))
    out["sv_max_rel_diff"] = float(np.max(np.abs(s - s_h) / s_h[0]))
    out["eig_max_rel_diff"] = float(np.max(np.abs(w - e_h.eigenvalues)) / e_h.eigenvalues[0])
print(json.dumps(out))
