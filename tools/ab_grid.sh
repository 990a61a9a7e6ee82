#!/usr/bin/env bash
# cfg4 / cfg5 quick benches under EM_GRID_SHORT values: tools/ab_grid.sh "v1 v2 ..."
for V in $1; do
  EM_GRID_SHORT=$V python -m paper_2409_03686_b200.build_native --force > /dev/null 2>&1
  for C in 4 5; do
    NR="--n-rep 100000"; [ $C -eq 5 ] && NR="--n-rep 50000"
    python bench.py --steps 10 --warmup 2 --config $C $NR --no-cpu-baseline 2>&1 | grep "^{" | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('GRID_SHORT=$V cfg$C', '%.4e' % d['value'])"
  done
done
python -m paper_2409_03686_b200.build_native --force > /dev/null 2>&1
