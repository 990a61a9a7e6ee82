#!/usr/bin/env bash
# Round measurement: tests, default bench, e2e breakdown, ncu launch list and
# one full ncu capture of the walk kernel (bench command, cfg2).
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
for C in 1 3 4 5; do
  timeout 300 python bench.py --config $C --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_${TAG}_c$C.log 2>&1
done
timeout 300 python tools/e2e_profile.py 2 > gpurun_out/e2e_$TAG.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 ; \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:walk_f32 -s 1 -c 1 \
   -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
tail -1 gpurun_out/pytest_$TAG.log; tail -1 gpurun_out/ncu_$TAG.log; cat gpurun_out/e2e_$TAG.log
