"""Executed warp instructions per CUDA source line (ncu source page, -lineinfo):
python tools/line_mix.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname = "?"
rows = []
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    ie = hdr.index("Instructions Executed")
    try:
        n = int(r[ie] or 0)
    except ValueError:
        continue
    if n:
        rows.append((n, fname, int(r[0]), r[1].strip()[:90]))
tot = sum(n for n, *_ in rows)
batches = None
print(f"total {tot:.4e}")
for n, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*n/tot:5.1f}% {n:12d} {f}:{ln:<5d} {src}")
by = {}
for n, f, ln, src in rows:
    by[f] = by.get(f, 0) + n
print({k: f"{100*v/tot:.1f}%" for k, v in by.items()})
