"""Debug: shell3d (3D ball with a concentric hole, max chain) counts per
build; prints row sums and step statistics for several walk counts."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2409_03686_b200 import backend as B  # noqa: E402
import test_gpu_parity as T  # noqa: E402

g = dict(np.load(ROOT / "tests" / "golden" / "cases.npz", allow_pickle=True))
gi, gf, cs, ks, poles, a0, a1 = T._frame_case(g, "shell3d")
print("gi", gi, "gf", gf, "cs", cs)
geom = B.GeomPack(gi, gf, cs)
s0 = B.SidePack(a0[0], a0[1], a0[2], 0, np.zeros(0), 2)
s1 = B.SidePack(a1[0], a1[1], a1[2], 0, np.zeros(0), 2)
out = {}
for n in (1000, 30000, 300000):
    with B.Plan(geom, ks, poles, 1e-5, 10**6, s0, s1, precision="fp32", chain="max") as plan:
        r = plan.run(4242, n)
    print(n, "row sums", r.counts.sum(1), "steps", r.steps_sum, "max", r.steps_max)
    out[str(n)] = r.counts
np.savez(sys.argv[1], **out)
