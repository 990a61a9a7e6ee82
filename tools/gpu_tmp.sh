set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sched.py tests/test_gpu_parity.py tests/test_gpu_edge.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_r2d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2d.log
for C in 3 4 5; do
 for S in auto persistent; do
  timeout 300 python bench.py --config $C --steps 5 --warmup 2 --no-cpu-baseline --sched $S > gpurun_out/bench_r2d_c${C}_$S.log 2>&1
 done
done
CMD="python bench.py --config 5 --steps 2 --warmup 1 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_r2d_c5.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_f32 -s 1 -c 1 -o /tmp/prof_r2d_c5 $CMD > gpurun_out/ncu_r2d_c5.log 2>&1
ncu -i /tmp/prof_r2d_c5.ncu-rep --page raw --csv > gpurun_out/raw_r2d_c5.csv 2>/dev/null
python tools/sass_mix.py /tmp/prof_r2d_c5.ncu-rep > gpurun_out/mix_r2d_c5.txt 2>&1
