#!/usr/bin/env python
"""Audit the built-in tuning table between its tuned orders: for every
GEMV row, time the table's choice (auto) against the stacked stream-K form
(shape 0, form 0; what the built-in rule picks for most orders) at three
orders spread over the row's range, and report rows where the table's
choice trails by more than 3 %.

    python scripts/table_audit.py [--min-order 2048]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1410_1726_b200 import tuner  # noqa: E402
from paper_1410_1726_b200.core import precision  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--min-order", type=int, default=2048)
ap.add_argument("--max-order", type=int, default=60000)
args = ap.parse_args()
doc = json.load(open(tuner.BUILTIN_TABLE))
kern = {"n": "gemv", "t": "gemv-t", "c": "gemv-c"}
for e in doc["entries"]:
    if e["op"] not in kern or e["n_hi"] < args.min_order or e["n_lo"] > args.max_order:
        continue
    lo, hi = max(e["n_lo"], args.min_order), min(e["n_hi"], args.max_order)
    sizes = sorted({int(round(math.exp(math.log(lo) + f * (math.log(hi) - math.log(lo))) / 32) * 32) for f in (0.15, 0.5, 0.85)})
    sizes = [s for s in sizes if lo <= s <= hi]
    if not sizes:
        continue
    k = kern[e["op"]]
    alt = tuner.TuneConfig(0, 0)
    pts = tuner.sweep(k, precision(e["prec"]), sizes, [tuner.auto_config(k), alt], reps=20, passes=2)
    worst = min(p0.measured_gbs / p1.measured_gbs for p0, p1 in
                ((next(p for p in pts if p.size == n and p.config.is_auto), next(p for p in pts if p.size == n and not p.config.is_auto)) for n in sizes))
    flag = "  <-- trails" if worst < 0.97 else ""
    print(json.dumps({"row": e, "sizes": sizes, "table_over_streamk_worst": round(worst, 3)}) + flag, flush=True)
