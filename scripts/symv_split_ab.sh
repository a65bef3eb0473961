#!/bin/bash
# Same-box A/B of the split SYMV schedule: the in-tree build with the tail
# grid (default share), the same build with KBLAS_SYMV_TAIL_PCT=0 (one
# grid), and optionally a previous build (ab_lib/lib_head.so), over
# scripts/ab_sweep_raw.py.  usage: bash scripts/symv_split_ab.sh OUT OPS SIZES
OUT=${1:-gpurun_out/symv_split_ab.jsonl}
OPS=${2:-dsymv,zhemv,ssymv,chemv}
SIZES=${3:-8192,16384,32768,65536}
: > $OUT
for rep in 1 2 3; do
  python scripts/ab_sweep_raw.py $PWD/paper_1410_1726_b200/libkblas_b200.so $OPS $SIZES split >> $OUT 2>&1
  KBLAS_SYMV_TAIL_PCT=0 python scripts/ab_sweep_raw.py $PWD/paper_1410_1726_b200/libkblas_b200.so $OPS $SIZES one >> $OUT 2>&1
  if [ -f ab_lib/lib_head.so ]; then
    python scripts/ab_sweep_raw.py $PWD/ab_lib/lib_head.so $OPS $SIZES head >> $OUT 2>&1
  fi
done
python - $OUT <<'PY'
import json, sys, statistics
rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
libs = sorted({r["lib"] for r in rows})
for k in sorted({(r["op"], r["n"]) for r in rows}):
    m = {L: statistics.median([r["gbs"] for r in rows if (r["op"], r["n"]) == k and r["lib"] == L]) for L in libs}
    print(k, m, "split/one %.3f" % (m["split"] / m["one"]), ("split/head %.3f" % (m["split"] / m["head"])) if "head" in m else "")
PY
