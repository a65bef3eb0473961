#!/bin/bash
# Same-box A/B: main kernels launched as programmatic dependents of the
# stream's previous kernel (KBLAS_PDL_CHAIN=1, default) or ordinarily (0),
# back-to-back device-vector calls (scripts/ab_sweep_raw.py).
OUT=${1:-gpurun_out/pdl_chain_ab.jsonl}
OPS=${2:-dgemv,dgemv_t,zgemv,sgemv,dsymv,ssymv,zhemv,chemv}
SIZES=${3:-1024,2048,4096,8192,16384}
L=$PWD/paper_1410_1726_b200/libkblas_b200.so
: > $OUT
for rep in 1 2 3; do
  for c in 0 1; do
    KBLAS_PDL_CHAIN=$c python scripts/ab_sweep_raw.py $L $OPS $SIZES chain$c >> $OUT 2>&1
  done
done
python3 - $OUT <<'PY'
import json, sys, statistics
rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
for k in sorted({(r["op"], r["n"]) for r in rows}):
    m = {L: statistics.median([r["gbs"] for r in rows if (r["op"], r["n"]) == k and r["lib"] == L]) for L in ("chain0", "chain1")}
    print(k, m, "chain1/chain0 %.3f" % (m["chain1"] / m["chain0"]))
PY
