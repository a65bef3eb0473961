OUT=gpurun_out/r2r_table_ab.jsonl
: > $OUT
S=1500,2300,3000,3900,4700,5500,6600,7700,9000,11000,14000,17000,20000,23000
for rep in 1 2; do
  python scripts/ab_sweep_raw.py $PWD/paper_1410_1726_b200/libkblas_b200.so dgemv,sgemv,cgemv,zgemv,dgemv_t,sgemv_t,cgemv_t,cgemv_c,zgemv_t,zgemv_c $S new >> $OUT 2>&1
  python scripts/ab_sweep_raw.py $PWD/ab_lib/lib_oldtable.so dgemv,sgemv,cgemv,zgemv,dgemv_t,sgemv_t,cgemv_t,cgemv_c,zgemv_t,zgemv_c $S old >> $OUT 2>&1
done
python3 - $OUT <<'PY'
import json, sys, statistics
rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
rat = []
worse = []
for k in sorted({(r["op"], r["n"]) for r in rows}):
    m = {L: statistics.median([r["gbs"] for r in rows if (r["op"], r["n"]) == k and r["lib"] == L]) for L in ("new", "old")}
    q = m["new"] / m["old"]
    rat.append(q)
    if q < 0.98 or q > 1.05:
        worse.append((k, round(m["new"]), round(m["old"]), round(q, 3)))
print("points", len(rat), "median new/old %.3f" % statistics.median(rat), "min %.3f max %.3f" % (min(rat), max(rat)))
print("geomean %.3f" % (statistics.geometric_mean(rat)))
for w in worse: print(w)
PY
