OUT=gpurun_out/r2n_split_scan.jsonl
: > $OUT
for rep in 1 2; do
for cfg in 0:4 4:4 6:2 6:4 8:4 10:4 8:8; do
  pct=${cfg%%:*}; kb=${cfg#*:}
  KBLAS_SYMV_TAIL_PCT=$pct KBLAS_SYMV_TAIL_ITEMS=$kb python scripts/ab_sweep_raw.py $PWD/paper_1410_1726_b200/libkblas_b200.so dsymv,zhemv,ssymv 16384,32768,65536 p${pct}k${kb} >> $OUT 2>&1
  KBLAS_SYMV_TAIL_PCT=$pct KBLAS_SYMV_TAIL_ITEMS=$kb python scripts/ab_sweep_raw.py $PWD/paper_1410_1726_b200/libkblas_b200.so dsymv 100000 p${pct}k${kb} >> $OUT 2>&1
done; done
python3 - <<PY
import json,statistics
rows=[json.loads(l) for l in open("$OUT") if l.startswith("{")]
libs=sorted({r["lib"] for r in rows}, key=lambda s:(int(s[1:s.index("k")]),int(s[s.index("k")+1:])))
for k in sorted({(r["op"],r["n"]) for r in rows}):
    m={L: statistics.median([r["gbs"] for r in rows if (r["op"],r["n"])==k and r["lib"]==L]) for L in libs}
    print(k, " ".join("%s:%.3f"%(L, m[L]/m["p0k4"]) for L in libs))
PY
