#!/usr/bin/env bash
# ncu full capture of the walk kernel for one config, summarised on the box:
#   tools/prof_cfg.sh TAG CFG NREP [extra bench args]   (KEEP=1 keeps the .ncu-rep)
TAG=$1; C=$2; NR=$3; shift 3
mkdir -p gpurun_out
CMD="python bench.py --config $C --n-rep $NR --steps 2 --warmup 1 --no-cpu-baseline $*"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_f32 -s 1 -c 1 \
   -o /tmp/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "$TAG ncu rc=$?"
python tools/sass_mix.py /tmp/prof_$TAG.ncu-rep > gpurun_out/mix_$TAG.txt 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>/dev/null
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv --print-source=sass > gpurun_out/sass_$TAG.csv 2>/dev/null
python tools/line_mix.py /tmp/prof_$TAG.ncu-rep 80 > gpurun_out/lines_$TAG.txt 2>&1
[ "$KEEP" = "1" ] && cp /tmp/prof_$TAG.ncu-rep gpurun_out/
true
