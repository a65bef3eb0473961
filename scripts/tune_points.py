#!/usr/bin/env python
"""Time explicit tuning-table candidates at explicit sizes (the tuner's
sweep, paper_1410_1726_b200.tuner.sweep) and print each against the
built-in choice.  For checking a table row the coarse/fine search did not
reach.

    python scripts/tune_points.py gemv-t d 24576,32768 0:-1,4:0,5:0
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1410_1726_b200 import tuner  # noqa: E402
from paper_1410_1726_b200.core import precision  # noqa: E402

kernel, tag = sys.argv[1], sys.argv[2]
sizes = [int(s) for s in sys.argv[3].split(",")]
cfgs = [tuner.auto_config(kernel)] + [tuner.TuneConfig(int(a), int(b)) for a, b in
                                      (c.split(":") for c in sys.argv[4].split(","))]
cfgs = list(dict.fromkeys(cfgs))
pts = tuner.sweep(kernel, precision(tag), sizes, cfgs, reps=20, passes=3)
for n in sizes:
    row = [p for p in pts if p.size == n]
    base = row[0].measured_gbs
    print(n, " ".join(f"{p.config.label()}:{p.measured_gbs:.0f}({p.measured_gbs / base:.3f})" for p in row), flush=True)
