#!/usr/bin/env bash
# One GPU iteration: gpu tests, bench, and an ncu profile of the walk kernel.
# usage: tools/gpu_cycle.sh TAG [bench args...]
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python bench.py --steps 20 --warmup 3 "$@" > gpurun_out/bench_$TAG.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline "$@" > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:walk_f32 -s 1 -c 1 \
  -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 1 --no-cpu-baseline "$@" > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
tail -2 gpurun_out/pytest_$TAG.log; tail -1 gpurun_out/ncu_$TAG.log
python - "$TAG" <<'PY'
import json, sys
tag = sys.argv[1]
for line in open(f"gpurun_out/bench_{tag}.log"):
    if line.startswith("{"):
        l = json.loads(line)
        print("value %.3e walks/s, steps/s %.3e, mean steps %.2f, ms/step %.3f, frac %.3f, e2e %.3e" % (
            l["value"], l["steps_per_s"], l["mean_steps_per_walk"], l["ms_per_step"],
            l["roofline"]["frac"], l["e2e"]["value"]))
PY
