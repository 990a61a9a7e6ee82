#!/usr/bin/env bash
# Final round-2 evidence run on the B200: the default bench (cfg3) and the
# reference arm, side benches, the ncu launch list of the bench command and
# one ncu --set full capture of the walk kernel per packed config.  Outputs
# under gpurun_out/ (tools/diag/collect_r2_final.py copies them to profiles/).
TAG=${1:-r2f}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_${TAG}_reference.log 2>&1; echo "reference rc=$?"
for C in 1 2 4 5; do
  timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c$C.log 2>&1
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --lanes one > gpurun_out/bench_${TAG}_c3_onewalk.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
for C in 3 2 4; do
  CMD="python bench.py --config $C --steps 2 --warmup 1 --no-cpu-baseline"
  timeout 300 $CMD > gpurun_out/plain_${TAG}_c$C.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_f32 -s 1 -c 1 \
     -o /tmp/prof_${TAG}_c$C $CMD > gpurun_out/ncu_${TAG}_c$C.log 2>&1
  echo "c$C ncu rc=$?"
  ncu -i /tmp/prof_${TAG}_c$C.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_c$C.csv 2>/dev/null
  python tools/ncu_metrics.py gpurun_out/raw_${TAG}_c$C.csv > gpurun_out/metrics_${TAG}_c$C.csv 2>&1
  python tools/sass_mix.py /tmp/prof_${TAG}_c$C.ncu-rep > gpurun_out/mix_${TAG}_c$C.txt 2>&1
  python tools/line_mix.py /tmp/prof_${TAG}_c$C.ncu-rep 60 > gpurun_out/lines_${TAG}_c$C.txt 2>&1
done
rm -f gpurun_out/raw_${TAG}_c*.csv
true
