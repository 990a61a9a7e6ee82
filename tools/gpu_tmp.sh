set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sched.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_analytic.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r2e.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2e.log
for C in 3 4 5; do
 for S in auto persistent pole-blocks; do
  timeout 300 python bench.py --config $C --steps 5 --warmup 2 --no-cpu-baseline --sched $S > gpurun_out/bench_r2e_c${C}_$S.log 2>&1
 done
done
timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2e_c2.log 2>&1
for C in 3 5; do
CMD="python bench.py --config $C --steps 2 --warmup 1 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_r2e_c$C.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_f32 -s 1 -c 1 -o /tmp/prof_r2e_c$C $CMD > gpurun_out/ncu_r2e_c$C.log 2>&1
ncu -i /tmp/prof_r2e_c$C.ncu-rep --page raw --csv > gpurun_out/raw_r2e_c$C.csv 2>/dev/null
python tools/sass_mix.py /tmp/prof_r2e_c$C.ncu-rep > gpurun_out/mix_r2e_c$C.txt 2>&1
python tools/line_mix.py /tmp/prof_r2e_c$C.ncu-rep 60 > gpurun_out/lines_r2e_c$C.txt 2>&1
done
