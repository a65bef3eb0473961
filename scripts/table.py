#!/usr/bin/env python
"""Render sweep JSONL files as an ops x sizes table: ours/cuBLAS GB/s."""
import json
import sys

rows = []
for f in sys.argv[1:]:
    rows += [json.loads(l) for l in open(f) if l.startswith("{")]
ops = []
for r in rows:
    if r["op"] not in ops:
        ops.append(r["op"])
sizes = sorted({r["n"] for r in rows})
print("| op | " + " | ".join(str(n) for n in sizes) + " |")
print("|---|" + "---|" * len(sizes))
for o in ops:
    cells = []
    for n in sizes:
        rr = [r for r in rows if r["op"] == o and r["n"] == n]
        if rr:
            r = rr[-1]
            c = f"{r['gbs']:.0f}"
            if "cublas_gbs" in r:
                c += f" / {r['cublas_gbs']:.0f}"
            cells.append(c)
        else:
            cells.append("")
    print(f"| {o} | " + " | ".join(cells) + " |")
