"""Refresh profiles/r01_cfg2_* from a profile_round.sh capture:
python tools/update_profiles.py TAG  (reads gpurun_out/{launches,prof}_TAG.*)"""
import csv
import io
import shutil
import subprocess
import sys
from pathlib import Path

root = Path(__file__).resolve().parents[1]
tag = sys.argv[1]
out = root / "gpurun_out"
prof = root / "profiles"
rep = out / f"prof_{tag}.ncu-rep"
shutil.copy(out / f"launches_{tag}.csv", prof / "r01_cfg2_launches.csv")
mix = subprocess.run([sys.executable, str(root / "tools" / "sass_mix.py"), str(rep)],
                     capture_output=True, text=True, check=True).stdout
(prof / "r01_cfg2_walk_f32_sass_mix.txt").write_text(mix)
raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
keys = ("gpu__time_duration", "dram__bytes", "inst_executed_pipe_", "issue_active",
        "warps_active", "registers_per_thread", "launch__grid_size", "launch__block_size",
        "thread_inst_executed_per_inst", "inst_executed.avg.per_cycle", "sm__inst_executed.sum",
        "lts__t_sectors_op", "warp_issue_stalled", "cycles_elapsed.avg.per_second",
        "occupancy")
with open(prof / "r01_cfg2_walk_f32_ncu_raw.csv", "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["metric", "value", "unit"])
    n = 0
    for h, u, v in zip(hdr, units, vals):
        if any(k in h for k in keys):
            w.writerow([h, v, u])
            n += 1
print(f"wrote {n} metrics")
raw_path = out / f"raw_{tag}.csv"
raw_path.write_text(raw)
subprocess.run([sys.executable, str(root / "tools" / "raw_summary.py"), str(raw_path)])
