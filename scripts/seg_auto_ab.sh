#!/bin/bash
# Same-box A/B: the wide SYMV kernel's split schedule with K = 12 where it
# keeps the split's rounds (default) against K = 6 (KBLAS_SYMV_SEG_AUTO=0).
OUT=${1:-gpurun_out/seg_auto_ab.jsonl}
L=$PWD/paper_1410_1726_b200/libkblas_b200.so
: > $OUT
for rep in 1 2 3; do
  for a in 0 1; do
    KBLAS_SYMV_SEG_AUTO=$a python scripts/ab_sweep_raw.py $L dsymv,zhemv,ssymv,chemv,dsymv_u 16384,24576,32768,49152,65536 auto$a >> $OUT 2>&1
  done
  for a in 0 1; do
    KBLAS_SYMV_SEG_AUTO=$a python scripts/ab_sweep_raw.py $L dsymv,zhemv 100000 auto$a >> $OUT 2>&1
  done
done
python3 - $OUT <<'PY'
import json, sys, statistics
rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
for k in sorted({(r["op"], r["n"]) for r in rows}):
    m = {L: statistics.median([r["gbs"] for r in rows if (r["op"], r["n"]) == k and r["lib"] == L]) for L in ("auto0", "auto1")}
    print(k, m, "auto/K6 %.3f" % (m["auto1"] / m["auto0"]))
PY
