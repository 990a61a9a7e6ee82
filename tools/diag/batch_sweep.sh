#!/usr/bin/env bash
# Rebuild with different steps-per-batch and bench cfg2/cfg3/cfg4 (max chain).
mkdir -p gpurun_out
for K in 4 8; do
  EM_BATCH_STEPS=$K python -m paper_2409_03686_b200.build_native --force > /dev/null 2>&1
  for C in 2 3 4; do
    NR=""; [ $C -ge 3 ] && NR="--n-rep 100000"
    timeout 300 python bench.py --steps 10 --warmup 2 --config $C $NR --no-cpu-baseline > gpurun_out/sweep_K${K}_c$C.log 2>&1
    python -c "
import json,sys
for l in open('gpurun_out/sweep_K${K}_c$C.log'):
    if l.startswith('{'):
        d=json.loads(l); print('K=$K cfg$C', '%.3e walks/s'%d['value'], '%.3e steps/s'%d['steps_per_s'], 'steps/walk %.2f'%d['mean_steps_per_walk'], 'frac %.3f'%d['roofline']['frac'])
"
  done
done
