#!/usr/bin/env bash
# GPU suite + full-size benches of cfg1..cfg5 (cfg2 = the default bench line)
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python bench.py > gpurun_out/bench_$TAG.log 2>&1
for C in 1 3 4 5; do
  timeout 300 python bench.py --config $C --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_${TAG}_c$C.log 2>&1
done
tail -1 gpurun_out/pytest_$TAG.log
for f in gpurun_out/bench_$TAG.log gpurun_out/bench_${TAG}_c*.log; do
  python -c "
import json, sys
for l in open('$f'):
    if l.startswith('{'):
        d = json.loads(l)
        print(d['config']['workload'][:14], d['config'].get('chain'), '%.3e' % d['value'], 'spw %.2f' % d['mean_steps_per_walk'], 'ms %.3f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'e2e %.3e' % d['e2e']['value'])
"
done
