#!/usr/bin/env python
"""Rebuild the built-in tuning table's GEMV rows below an order from dense
tuning points (scripts/tune_dense.py, two runs per job), keeping every
other row (SYMV/HEMV, GEMV above the dense range, clipped to start there).

A dense size gets a row only if one candidate beat the bare built-in rule
by >= --min-gain in BOTH runs (the candidate with the largest worst-run
gain wins).  Each size covers the orders nearest to it on a log scale.

    python scripts/merge_dense.py --top 24576 --inc ... --json ... a1.csv:b1.csv a2.csv:b2.csv ...
"""
import argparse
import csv
import json
import math
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read(path):
    out = defaultdict(dict)  # (kernel, prec, size) -> {(shape, form, waves): gbs}
    for r in csv.DictReader(open(path)):
        key = (r["kernel"], r["precision"], int(r["size"]))
        out[key][(int(r["shape"]), int(r["form"]), int(r["waves"]))] = float(r["measured_gbs"])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("pairs", nargs="+", help="runA.csv:runB.csv per job")
    ap.add_argument("--top", type=int, default=24576, help="dense rows cover orders below this")
    ap.add_argument("--bottom", type=int, default=724)
    ap.add_argument("--min-gain", type=float, default=0.02)
    ap.add_argument("--json", required=True)
    ap.add_argument("--inc", required=True)
    args = ap.parse_args()
    opmap = {"gemv": "n", "gemv-t": "t", "gemv-c": "c"}
    new_rows, jobs = [], set()
    for pair in args.pairs:
        a, b = (read(p) for p in pair.split(":"))
        keys = sorted(set(a) & set(b), key=lambda k: k[2])
        if not keys:
            continue
        kernel, tag = keys[0][0], keys[0][1]
        op = opmap[kernel]
        jobs.add((tag, op))
        auto = (0, -1, 0)
        sizes = [k[2] for k in keys]
        for i, k in enumerate(keys):
            n = k[2]
            ca, cb = a[k], b[k]
            best, gain = None, 0.0
            for cfg in set(ca) & set(cb):
                if cfg == auto or auto not in ca or auto not in cb:
                    continue
                g = min(ca[cfg] / ca[auto], cb[cfg] / cb[auto]) - 1
                if g >= args.min_gain and g > gain:
                    best, gain = cfg, g
            if best is None:
                continue
            lo = args.bottom if i == 0 else math.floor(math.sqrt(sizes[i - 1] * n)) + 1
            hi = args.top - 1 if i == len(sizes) - 1 else math.floor(math.sqrt(n * sizes[i + 1]))
            hi = min(hi, args.top - 1)
            if lo > hi:
                continue
            new_rows.append({"prec": tag, "op": op, "n_lo": lo, "n_hi": hi, "shape": best[0], "form": best[1],
                             "waves": best[2], "_gain": gain, "_n": n})
    old = json.load(open(os.path.join(ROOT, "paper_1410_1726_b200", "tuning", "b200.json")))["entries"]
    kept = []
    for e in old:
        if (e["prec"], e["op"]) in jobs:
            if e["n_hi"] < args.top:
                continue  # replaced by the dense rows
            e = dict(e, n_lo=max(e["n_lo"], args.top))
        kept.append(e)
    rows = kept + [{k: v for k, v in r.items() if not k.startswith("_")} for r in new_rows]
    order = {"n": 0, "t": 1, "c": 2, "l": 3, "u": 4}
    rows.sort(key=lambda e: (order[e["op"]], e["prec"], e["n_lo"]))
    by = defaultdict(list)
    for e in rows:
        by[(e["prec"], e["op"])].append((e["n_lo"], e["n_hi"]))
    for k, rs in by.items():
        rs.sort()
        assert all(x[1] < y[0] for x, y in zip(rs, rs[1:])), (k, rs)
    json.dump({"format": "kblas-b200-tuning/1", "device": "NVIDIA B200", "entries": rows}, open(args.json, "w"),
              indent=1)
    with open(args.inc, "w") as fh:
        fh.write("// Built-in tuning table (NVIDIA B200).  GEMV rows below order "
                 f"{args.top}: scripts/merge_dense.py over\n")
        fh.write("// dense tuning points (scripts/tune_dense.py, two runs, a row only where one config beat the\n")
        fh.write(f"// bare rules by >= {100 * args.min_gain:.0f} % in both; profiles/r2r_dense_*.csv).  Other rows: "
                 "scripts/merge_tuning.py over\n")
        fh.write("// profiles/r1z_tune_points2_{a,b}.csv and the round-2 point checks (DESIGN.md section 7.1).\n")
        fh.write("// {prec, op, n_lo, n_hi, shape, form, waves}\n")
        for e in rows:
            fh.write(f"{{'{e['prec']}', '{e['op']}', {e['n_lo']}, {e['n_hi']}, {e['shape']}, {e['form']}, {e['waves']}}},\n")
    print(f"{len(rows)} rows ({len(new_rows)} dense, {len(kept)} kept)")
    for r in new_rows:
        print(f"  {r['prec']} {r['op']} {r['n_lo']:6d}-{r['n_hi']:6d} (n={r['_n']}): shape={r['shape']} form={r['form']} "
              f"+{100 * r['_gain']:.1f} %")


if __name__ == "__main__":
    main()
