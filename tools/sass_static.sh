#!/bin/bash
# Static SASS of one walk_f32 instantiation (default: cfg2's kernel) for quick
# before/after comparisons without a GPU:  tools/sass_static.sh [mangled-name-substring]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
K=${1:-walk_f32_kernelILi2ELi1ELi0ELi1ELb0ELi0ELi2ELi0E}
OUT=${OUT:-/tmp/sass_static}
mkdir -p $OUT
/usr/local/cuda/bin/nvcc -cubin -o $OUT/walk_f32.cubin $ROOT/paper_2409_03686_b200/csrc/walk_f32.cu \
  -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I $ROOT/include \
  -fmad=true -prec-sqrt=false -prec-div=false -DEM_BATCH_STEPS=${EM_BATCH_STEPS:-8} \
  -DEM_MIN_BLOCKS=${EM_MIN_BLOCKS:-0} -DEM_ANGLE_BITS=${EM_ANGLE_BITS:-16} -Xptxas -v 2> $OUT/ptxas.log
/usr/local/cuda/bin/cuobjdump -sass $OUT/walk_f32.cubin > $OUT/all.sass
python3 - "$OUT" "$K" <<'PY'
import re, sys
out, k = sys.argv[1], sys.argv[2]
s = open(f"{out}/all.sass").read()
i = s.index("Function : ", s.index(k) - 200)
i = s.rfind("Function : ", 0, s.index(k) + 1)
j = s.find("Function :", i + 10)
body = s[i:j if j > 0 else None]
ins = [l for l in body.splitlines() if re.search(r"/\*[0-9a-f]{4,}\*/", l)]
ins = [re.sub(r"/\* 0x[0-9a-f]+ \*/", "", l).strip() for l in ins]
open(f"{out}/kernel.txt", "w").write("\n".join(ins))
print(body.splitlines()[0].strip(), "instructions:", len(ins))
PY
grep -A2 "$K" $OUT/ptxas.log | grep -o "Used [0-9]* registers" | head -1
