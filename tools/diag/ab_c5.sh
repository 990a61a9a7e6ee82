#!/usr/bin/env bash
# cfg5 / cfg2 quick benches under compile-time knob values: tools/ab_c5.sh VAR "v1 v2"
VAR=$1; VALS=$2
mkdir -p gpurun_out
for V in $VALS; do
  env $VAR=$V python -m paper_2409_03686_b200.build_native --force > /dev/null 2>&1
  for C in 5 2; do
    NR=""; [ $C -eq 5 ] && NR="--n-rep 100000"
    timeout 300 python bench.py --steps 10 --warmup 2 --config $C $NR --no-cpu-baseline > gpurun_out/ab5_${V}_c$C.log 2>&1
    python -c "
import json
for l in open('gpurun_out/ab5_${V}_c$C.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$VAR=$V cfg$C', '%.3e walks/s'%d['value'], 'steps/walk %.2f'%d['mean_steps_per_walk'], 'ms %.3f'%d['ms_per_step'])
"
  done
done
python -m paper_2409_03686_b200.build_native --force > /dev/null 2>&1
