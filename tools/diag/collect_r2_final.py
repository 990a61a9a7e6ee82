"""Copy a tools/gpu_r2_final.sh run (gpurun_out/*_TAG*) into profiles/r02_*:
python tools/diag/collect_r2_final.py TAG"""
import json
import shutil
import sys
from pathlib import Path

root = Path(__file__).resolve().parents[2]
out, prof = root / "gpurun_out", root / "profiles"
tag = sys.argv[1]


def line(path):
    for l in open(path):
        if l.startswith("{"):
            return l
    raise SystemExit(f"no JSON line in {path}")


for c in (2, 3, 4):
    shutil.copy(out / f"metrics_{tag}_c{c}.csv", prof / f"r02_cfg{c}_walk_f32_ncu_metrics.csv")
    shutil.copy(out / f"mix_{tag}_c{c}.txt", prof / f"r02_cfg{c}_walk_f32_sass_mix.txt")
    shutil.copy(out / f"lines_{tag}_c{c}.txt", prof / f"r02_cfg{c}_walk_f32_lines.txt")
(prof / "r02_bench_cfg3.json.log").write_text(line(out / f"bench_{tag}.log"))
(prof / "r02_bench_cfg3_reference.json.log").write_text(line(out / f"bench_{tag}_reference.log"))
(prof / "r02_cfg3_launches.csv").write_text(
    "".join(l for l in open(out / f"launches_{tag}.csv") if not l.startswith("==")))
rows = ["# round-2 final build, one B200: python bench.py [--config C --steps 10 --warmup 3] "
        "(tools/gpu_r2_final.sh)"]
for f, name in ((f"bench_{tag}.log", "cfg3 (default bench)"),
                (f"bench_{tag}_c3_onewalk.log", "cfg3 --lanes one (one-walk-per-lane kernel; e2e goes "
                                                "through the plugin = packed)"),
                (f"bench_{tag}_c1.log", "cfg1"), (f"bench_{tag}_c2.log", "cfg2"),
                (f"bench_{tag}_c4.log", "cfg4"), (f"bench_{tag}_c5.log", "cfg5")):
    d = json.loads(line(out / f))
    rows.append("%s: %.4e walks/s, e2e %.4e, steps/walk %.4f, kernel %.3f ms, walks/lane %s, "
                "scheduler %s, FP32 frac %.3f, clocks %s MHz %s"
                % (name, d["value"], d["e2e"]["value"], d["mean_steps_per_walk"],
                   d["roofline"]["kernel_ms"], d["config"].get("walks_per_lane"),
                   d["config"].get("scheduler"), d["roofline"]["frac"], d["clocks"]["sm_mhz"],
                   d["clocks"]["reasons"]))
d = json.loads(line(out / f"bench_{tag}_reference.log"))
rows.append("cfg3 --impl reference: %.4e walks/s (%s)" % (d["value"], d["cpu_baseline"]["sample"]))
(prof / "r02_bench_all.txt").write_text("\n".join(rows) + "\n")
for f in ("cfg2_full", "cfg2_sigma", "cfg2_u1", "cfg3_64x1e6_vs_1e5", "cfg4_64x1e6_vs_1e5",
          "cfg5_64x1e6_vs_1e5"):
    if (out / f"fullscale_{f}.json").exists():
        shutil.copy(out / f"fullscale_{f}.json", prof / f"r02_fullscale_{f}.json")
if (out / "refsuite.log").exists():
    shutil.copy(out / "refsuite.log", prof / "r02_refsuite.txt")
print("\n".join(rows))
