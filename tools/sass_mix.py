"""Per-opcode instruction mix of the hot region of a kernel from an ncu
report's source page (SASS): python tools/sass_mix.py report.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ia = hdr.index("Instructions Executed")
isrc = hdr.index("Source")
iavg = hdr.index("Avg. Threads Executed")
ist = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ia] or 0) for r in data)
base = max(int(r[ia] or 0) for r in data if "IMAD.WIDE.U32" in r[isrc]) if any("IMAD.WIDE.U32" in r[isrc] for r in data) else 1
print(f"total warp instructions {tot:.4g}; batch count (Philox IMAD.WIDE) {base:.4g}; "
      f"instr per batch {tot / base:.1f}")
ops = collections.Counter()
lanes = 0.0
for r in data:
    n = int(r[ia] or 0)
    s = r[isrc].split()
    op = s[1] if s and s[0].startswith("@") else (s[0] if s else "?")
    ops[op.split(".")[0]] += n
    lanes += n * float(r[iavg] or 0)
print(f"avg active lanes {lanes / tot:.2f}")
for op, n in ops.most_common(30):
    print(f"  {op:10s} {n / base:7.1f}/batch  {100 * n / tot:5.1f}%")
# stall samples by line
st = sorted(((int(r[ist] or 0), r[isrc][:80], int(r[ia] or 0)) for r in data), reverse=True)[:15]
print("top stall lines:")
for s_, src, n in st:
    print(f"  {s_:6d} exec {n:10d}  {src}")
