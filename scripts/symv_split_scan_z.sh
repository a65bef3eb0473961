OUT=gpurun_out/r2p_z_split_scan.jsonl
: > $OUT
L=$PWD/paper_1410_1726_b200/libkblas_b200.so
for rep in 1 2 3; do
for cfg in 0:4 3:4 6:4 6:8 10:8; do
  pct=${cfg%%:*}; kb=${cfg#*:}
  KBLAS_SYMV_TAIL_PCT=$pct KBLAS_SYMV_TAIL_ITEMS=$kb python scripts/ab_sweep_raw.py $L zhemv 100000 p${pct}k${kb} >> $OUT 2>&1
  KBLAS_SYMV_TAIL_PCT=$pct KBLAS_SYMV_TAIL_ITEMS=$kb python scripts/ab_sweep_raw.py $L zhemv,chemv 49152 p${pct}k${kb} >> $OUT 2>&1
done; done
python3 - <<PY
import json,statistics
rows=[json.loads(l) for l in open("$OUT") if l.startswith("{")]
libs=["p0k4","p3k4","p6k4","p6k8","p10k8"]
for k in sorted({(r["op"],r["n"]) for r in rows}):
    m={L: statistics.median([r["gbs"] for r in rows if (r["op"],r["n"])==k and r["lib"]==L]) for L in libs}
    print(k, " ".join("%s:%.1f(%.3f)"%(L, m[L], m[L]/m["p0k4"]) for L in libs))
PY
