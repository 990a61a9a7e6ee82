#!/usr/bin/env bash
# A/B a compile-time knob: tools/ab_bench.sh VAR "v1 v2"  (benches cfg2..cfg5)
VAR=$1; VALS=$2
mkdir -p gpurun_out
for V in $VALS; do
  env EXITMEASURE_B200_KNOBS=1 $VAR=$V python -m paper_2409_03686_b200.build_native --force > /dev/null 2>&1
  for C in 2 3 4 5; do
    NR=""; [ $C -ge 3 ] && NR="--n-rep 100000"; [ $C -eq 5 ] && NR="--n-rep 20000"
    timeout 300 python bench.py --steps 10 --warmup 2 --config $C $NR --no-cpu-baseline > gpurun_out/ab_${V}_c$C.log 2>&1
    python -c "
import json
for l in open('gpurun_out/ab_${V}_c$C.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$VAR=$V cfg$C', '%.3e walks/s'%d['value'], 'steps/walk %.2f'%d['mean_steps_per_walk'], 'frac %.3f'%d['roofline']['frac'])
"
  done
done
python -m paper_2409_03686_b200.build_native --force > /dev/null 2>&1
