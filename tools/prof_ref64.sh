#!/usr/bin/env bash
# ncu capture of the REF64 walk kernel (cfg2, reduced walks), summarised on the box
mkdir -p gpurun_out
CMD="python bench.py --config 2 --n-rep 20000 --precision ref64 --steps 1 --warmup 1 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_ref64.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_ref64 -s 1 -c 1 \
   -o /tmp/prof_ref64 $CMD > gpurun_out/ncu_ref64.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_ref64.ncu-rep --page raw --csv > gpurun_out/raw_ref64.csv 2>/dev/null
python tools/line_mix.py /tmp/prof_ref64.ncu-rep 50 > gpurun_out/lines_ref64.txt 2>&1
python tools/sass_mix.py /tmp/prof_ref64.ncu-rep > gpurun_out/mix_ref64.txt 2>&1
