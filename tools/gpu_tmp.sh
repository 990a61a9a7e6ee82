mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rfE > gpurun_out/pytest_r2f.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2f.log
tail -3 gpurun_out/pytest_r2f.log
timeout 600 python bench.py > gpurun_out/bench_r2f.log 2>&1
for C in 2 4 5; do timeout 300 python bench.py --config $C --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_r2f_c$C.log 2>&1; done
CMD="python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_r2f_c3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_f32 -s 1 -c 1 -o /tmp/prof_r2f_c3 $CMD > gpurun_out/ncu_r2f_c3.log 2>&1
ncu -i /tmp/prof_r2f_c3.ncu-rep --page raw --csv > gpurun_out/raw_r2f_c3.csv 2>/dev/null
python tools/sass_mix.py /tmp/prof_r2f_c3.ncu-rep > gpurun_out/mix_r2f_c3.txt 2>&1
python tools/line_mix.py /tmp/prof_r2f_c3.ncu-rep 400 > gpurun_out/lines_r2f_c3.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2f_c3.csv $CMD > gpurun_out/ncu_launch_r2f.log 2>&1
