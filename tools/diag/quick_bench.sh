#!/usr/bin/env bash
# gpu parity tests (-x) + short benches of cfg2..cfg5 (reduced walks for 3..5)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/qb_pytest.log 2>&1; tail -1 gpurun_out/qb_pytest.log
for C in 2 3 4 5; do
  NR=""; [ $C -ge 3 ] && NR="--n-rep 100000"; [ $C -eq 5 ] && NR="--n-rep 20000"
  timeout 300 python bench.py --steps 10 --warmup 2 --config $C $NR --no-cpu-baseline "$@" > gpurun_out/qb_c$C.log 2>&1
  python -c "
import json
for l in open('gpurun_out/qb_c$C.log'):
    if l.startswith('{'):
        d=json.loads(l); print('cfg$C', '%.3e walks/s'%d['value'], '%.3e steps/s'%d['steps_per_s'], 'steps/walk %.2f'%d['mean_steps_per_walk'], 'frac %.3f'%d['roofline']['frac'])
"
done
