mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_plugin.py tests/test_gpu_refsuite.py tests/test_gpu_edge.py -m gpu -q -p no:cacheprovider -rfE > gpurun_out/pytest_r2h.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2h.log
tail -3 gpurun_out/pytest_r2h.log
for C in 2 4; do
CMD="python bench.py --config $C --steps 2 --warmup 1 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_r2h_c$C.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_f32 -s 1 -c 1 -o /tmp/prof_r2h_c$C $CMD > gpurun_out/ncu_r2h_c$C.log 2>&1
ncu -i /tmp/prof_r2h_c$C.ncu-rep --page raw --csv > gpurun_out/raw_r2h_c$C.csv 2>/dev/null
python tools/sass_mix.py /tmp/prof_r2h_c$C.ncu-rep > gpurun_out/mix_r2h_c$C.txt 2>&1
python tools/line_mix.py /tmp/prof_r2h_c$C.ncu-rep 400 > gpurun_out/lines_r2h_c$C.txt 2>&1
done
