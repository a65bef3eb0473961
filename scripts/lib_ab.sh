#!/bin/bash
# Same-box A/B of two library builds over scripts/sweep.py: the in-tree
# build against ab_lib/libkblas_b200_prev.so (KBLAS_LIB), interleaved.
# usage: bash scripts/lib_ab.sh OPS SIZES OUT
OPS=${1:-dsymv,ssymv,chemv}
SIZES=${2:-4096,8192,12288}
OUT=${3:-gpurun_out/lib_ab.jsonl}
: > $OUT
for rep in 1 2 3; do
  for v in cur prev; do
    if [ $v = prev ]; then export KBLAS_LIB=$PWD/ab_lib/libkblas_b200_prev.so; else unset KBLAS_LIB; fi
    timeout 600 python scripts/sweep.py --ops $OPS --sizes $SIZES --no-cublas --passes 2 2>/dev/null \
      | python -c "import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(json.dumps({'lib':'$v','rep':$rep,'op':d['op'],'n':d['n'],'gbs':d['gbs']}))" >> $OUT
  done
done
unset KBLAS_LIB
python - $OUT <<'PY'
import json, sys, statistics
rows = [json.loads(l) for l in open(sys.argv[1])]
keys = sorted({(r["op"], r["n"]) for r in rows})
for k in keys:
    c = [r["gbs"] for r in rows if (r["op"], r["n"]) == k and r["lib"] == "cur"]
    p = [r["gbs"] for r in rows if (r["op"], r["n"]) == k and r["lib"] == "prev"]
    print(k, "cur", c, "prev", p, "cur/prev %.3f" % (statistics.median(c) / statistics.median(p)))
PY
