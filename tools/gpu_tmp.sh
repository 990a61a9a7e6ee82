mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rfE > gpurun_out/pytest_r2g.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2g.log
tail -3 gpurun_out/pytest_r2g.log
timeout 600 python bench.py > gpurun_out/bench_r2g.log 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_r2g_ref.log 2>&1
tail -1 gpurun_out/bench_r2g.log | cut -c1-400
