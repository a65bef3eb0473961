#!/usr/bin/env python
"""Run the measured coarse/fine tuner (paper_1410_1726_b200.tuner) over
every kernel and precision and save one tuning table.

    python scripts/tune_all.py --sizes 1024,...,49152 --save table.json --points points.csv

One JSON line per (kernel, precision, uplo) on stdout: the coarse winner
and, per size, the fine winner with its GB/s against the built-in
choice's.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1410_1726_b200 import tuner  # noqa: E402

JOBS = [("gemv", t, "l") for t in "sdcz"] + [("gemv-t", t, "l") for t in "sdcz"] + \
       [("gemv-c", t, "l") for t in "cz"] + \
       [(k, t, u) for k, t in (("symv", "s"), ("symv", "d"), ("hemv", "c"), ("hemv", "z")) for u in "lu"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1024,2048,4096,8192,12288,16384,24576,32768,49152")
    ap.add_argument("--jobs", default=None, help="comma list of kernel:prec[:uplo]")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--min-gain", type=float, default=0.02)
    ap.add_argument("--save", required=True)
    ap.add_argument("--points", default=None)
    ap.add_argument("--keep-table", action="store_true",
                    help="measure against the library's built-in table instead of the bare rules")
    args = ap.parse_args()
    sizes = [int(s) for s in args.sizes.split(",")]
    jobs = JOBS
    if args.jobs:
        jobs = []
        for j in args.jobs.split(","):
            parts = j.split(":")
            jobs.append((parts[0], parts[1], parts[2] if len(parts) > 2 else "l"))
    if not args.keep_table:
        tuner.clear()
    allpts = []
    for kernel, tag, uplo in jobs:
        coarse, fine = tuner.tune(kernel, tag, sizes, uplo=uplo, reps=args.reps, min_gain=args.min_gain)
        rows = tuner.entries_for(fine) if args.keep_table else tuner.apply(fine)
        allpts += coarse.points + fine.points
        per = {}
        for n in sizes:
            pts = [p for p in fine.points if p.size == n]
            win = fine.per_size[n]
            wp = next(p for p in pts if p.config == win)
            per[n] = {"winner": win.label(), "gbs": round(wp.measured_gbs, 1),
                      "builtin_gbs": round(pts[0].measured_gbs, 1),
                      "best_any": round(max(p.measured_gbs for p in pts), 1)}
        print(json.dumps({"kernel": kernel, "prec": tag, "uplo": uplo, "coarse": coarse.winner.label(),
                          "coarse_points": {p.config.label(): round(p.measured_gbs, 1) for p in coarse.points},
                          "rows": len(rows), "per_size": per}), flush=True)
    tuner.save(args.save, device=torch.cuda.get_device_name())
    if args.points:
        with open(args.points, "w", newline="") as fh:
            tuner.write_sweep_csv(allpts, fh)


if __name__ == "__main__":
    main()
