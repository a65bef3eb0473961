#!/bin/bash
# Same-box A/B of two builds of the library with scripts/sweep.py (no
# cuBLAS): the working tree's build against one prepared under _alt/
# (a copy of paper_1410_1726_b200/ with its built .so, bench.py,
# scripts/sweep.py and oracle/ from the other revision; _alt/ is
# git-ignored but travels with gpurun).  Used for the x-load change
# (coherent loads instead of ld.global.nc, profiles/r2f_xload_ab.txt).
mkdir -p gpurun_out
OPS=${OPS:-dgemv,cgemv,dgemv_t,cgemv_c,zgemv_t,dsymv,ssymv,zhemv,sgemv_t}
SZ=${SZ:-2048,4096,8192,16384}
for rep in 1 2; do
  timeout 400 python scripts/sweep.py --no-cublas --ops $OPS --sizes $SZ --out gpurun_out/ab_new_$rep.jsonl > /dev/null 2>&1
  (cd _alt && timeout 400 python scripts/sweep.py --no-cublas --ops $OPS --sizes $SZ --out ../gpurun_out/ab_old_$rep.jsonl > /dev/null 2>&1)
done
python - <<'PY'
import json, collections
def load(tag):
    d = collections.defaultdict(list)
    for rep in (1, 2):
        for l in open(f"gpurun_out/ab_{tag}_{rep}.jsonl"):
            r = json.loads(l); d[(r["op"], r["n"])].append(r["gbs"])
    return {k: max(v) for k, v in d.items()}
new, old = load("new"), load("old")
for k in sorted(new):
    print(k, round(new[k]), round(old[k]), round(new[k] / old[k], 3))
PY
