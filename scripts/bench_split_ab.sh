#!/bin/bash
# bench.py (configs[4] headline, ZHEMV 100k, configs[1]) with the split
# SYMV schedule (default) and with one grid (KBLAS_SYMV_TAIL_PCT=0),
# interleaved on one box.
OUT=${1:-gpurun_out/bench_split_ab.jsonl}
: > $OUT
for rep in 1 2; do
  for pct in 0 6; do
    KBLAS_SYMV_TAIL_PCT=$pct timeout 600 python bench.py --no-cpu --steps 30 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); z=d['zhemv_100k']; c1=d['configs1_dsymv_32768']
print(json.dumps({'tail_pct':$pct,'rep':$rep,'d100k':d['value'],'d100k_kernel_gbs':d['roofline']['achieved'],'e2e':d['e2e']['value'],
 'z100k':z['value'],'c1':c1['value'],'c1_kernel_gbs':c1['roofline']['achieved'],'plan':d['plan']}))" >> $OUT
  done
done
cat $OUT
