"""CPU reference timing beside the GPU numbers: the reference's
own run_accumulate (oracle/_ref; the C restatement for cfg5) at threads=1 and
threads=os.cpu_count(), at two walk counts each (walks are iid, so time must
be linear in N).  Prints one JSON line; run on the GPU box's host.
python tools/cpu_scan.py [cfg ...]"""
import json
import os
import platform
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2409_03686_b200 import configs  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


cfgs = [int(c) for c in sys.argv[1:]] or [1, 2, 3, 4, 5]
allt = os.cpu_count() or 1
out = {"cpu_model": cpu_model(), "cpu_count": allt, "runs": []}
for c in cfgs:
    cfg = configs.get(c)
    base = bench.REF_SAMPLE[c]
    for threads, n in ((1, max(base // 16, 4)), (1, max(base // 8, 8)), (allt, base), (allt, 2 * base)):
        wps, sps, kind, dt, spw = bench.cpu_reference_walks_per_s(cfg, n, threads)
        out["runs"].append({"cfg": c, "threads": threads, "walks_per_pole": n,
                            "walks": cfg.n_poles * n, "seconds": dt, "walks_per_s": wps,
                            "steps_per_s": sps, "steps_per_walk": spw, "kind": kind})
        print(f"cfg{c} threads={threads} n={n}: {wps:.3e} walks/s ({dt:.2f} s, {kind})",
              file=sys.stderr, flush=True)
print(json.dumps(out))
