#!/usr/bin/env bash
# Round-2 GPU iteration: gpu tests, the default bench (cfg3) and cfg2, then
# ncu captures of the walk kernel for the configs given (raw/sass/line CSVs
# only: the .ncu-rep stays in /tmp so gpurun_out/ stays under its cap).
#   tools/gpu_r2.sh TAG "3 5"      (PYTEST=0 skips the test suite)
TAG=$1; CFGS=${2:-}
mkdir -p gpurun_out
if [ "${PYTEST:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/pytest_$TAG.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log; tail -3 gpurun_out/pytest_$TAG.log
fi
if [ "${BENCH:-1}" = "1" ]; then
  timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
  timeout 300 python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench_${TAG}_c2.log 2>&1
  tail -1 gpurun_out/bench_$TAG.log
fi
for C in $CFGS; do
  CMD="python bench.py --config $C --steps 2 --warmup 1 --no-cpu-baseline"
  timeout 300 $CMD > gpurun_out/plain_${TAG}_c$C.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_f32 -s 1 -c 1 \
     -o /tmp/prof_${TAG}_c$C $CMD > gpurun_out/ncu_${TAG}_c$C.log 2>&1
  echo "c$C ncu rc=$?"
  ncu -i /tmp/prof_${TAG}_c$C.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_c$C.csv 2>/dev/null
  ncu -i /tmp/prof_${TAG}_c$C.ncu-rep --page source --csv --print-source=sass > gpurun_out/sass_${TAG}_c$C.csv 2>/dev/null
  python tools/sass_mix.py /tmp/prof_${TAG}_c$C.ncu-rep > gpurun_out/mix_${TAG}_c$C.txt 2>&1
  python tools/line_mix.py /tmp/prof_${TAG}_c$C.ncu-rep 80 > gpurun_out/lines_${TAG}_c$C.txt 2>&1
done
true
