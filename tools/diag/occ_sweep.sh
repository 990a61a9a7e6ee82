#!/usr/bin/env bash
# Rebuild the FP32 kernel at several occupancy targets and bench cfg2..cfg5.
mkdir -p gpurun_out
for MB in 4 5 6; do
  EM_MIN_BLOCKS=$MB python -m paper_2409_03686_b200.build_native --force --verbose > gpurun_out/build_mb$MB.log 2>&1
  grep -c "spill stores" gpurun_out/build_mb$MB.log > /dev/null
  for C in 2 3 4 5; do
    NR=""; [ $C -ge 3 ] && NR="--n-rep 100000"; [ $C -eq 5 ] && NR="--n-rep 20000"
    timeout 300 python bench.py --steps 10 --warmup 2 --config $C $NR --no-cpu-baseline > gpurun_out/occ_mb${MB}_c$C.log 2>&1
    python -c "
import json
for l in open('gpurun_out/occ_mb${MB}_c$C.log'):
    if l.startswith('{'):
        d=json.loads(l); print('MB=$MB cfg$C', '%.3e walks/s'%d['value'], '%.3e steps/s'%d['steps_per_s'], 'frac %.3f'%d['roofline']['frac'])
"
  done
done
EM_MIN_BLOCKS=4 python -m paper_2409_03686_b200.build_native --force > /dev/null 2>&1
