#!/usr/bin/env bash
# tools/diag/ab_libs.sh CFG "tag1 tag2 ..."  -- bench each variants/lib_<tag>.so ("prod" = the in-tree library)
CFG=$1; TAGS=$2; EXTRA=${3:-}
mkdir -p gpurun_out
for T in $TAGS; do
  if [ "$T" = "prod" ]; then unset EXITMEASURE_B200_LIB; else export EXITMEASURE_B200_LIB=variants/lib_$T.so; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --config $CFG --no-cpu-baseline $EXTRA > gpurun_out/abl_${T}_c$CFG.log 2>&1
  python - <<PY
import json
for l in open('gpurun_out/abl_${T}_c$CFG.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$T cfg$CFG', '%.4e walks/s'%d['value'], 'e2e %.4e'%d['e2e']['value'], 'steps/walk %.3f'%d['mean_steps_per_walk'], 'kernel ms %.3f' % d['roofline'].get('kernel_ms', 0))
PY
done
