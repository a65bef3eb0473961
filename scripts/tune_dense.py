#!/usr/bin/env python
"""Dense tuning points for one GEMV kernel: every candidate of an
explicit list at geometrically spaced orders (the built-in table was
tuned at octave-spaced orders, and between them a row can be far from the
best choice: ZGEMV-N 4864 ran the cluster split form at 4.8 TB/s where
stream-K gives 6.0).  Writes tuner.write_sweep_csv points, measured against
the bare built-in rules (table cleared).

    python scripts/tune_dense.py gemv d 1024 24576 8 OUT.csv
      (kernel, precision, lowest order, highest order, steps per octave)
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1410_1726_b200 import tuner  # noqa: E402
from paper_1410_1726_b200.core import precision  # noqa: E402

kernel, tag, lo, hi, per_oct, out = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), sys.argv[6]
sizes = []
k = 0
while True:
    n = int(round(lo * 2 ** (k / per_oct) / 32) * 32)
    if n > hi:
        break
    if not sizes or n != sizes[-1]:
        sizes.append(n)
    k += 1
op = tuner.op_of(kernel)
cands = [tuner.auto_config(kernel)]
if op == "n":
    cands += [tuner.TuneConfig(s, f) for s in (0, 3, 4, 5) for f in (-1, 0, 1, 2) if (s, f) != (0, -1)]
    cands += [tuner.TuneConfig(s, 3) for s in tuner.ROWOWN_SHAPES]
else:
    cands += [tuner.TuneConfig(s, f) for s in (0, 3, 4, 5) for f in (-1, 0, 1) if (s, f) != (0, -1)]
tuner.clear()
pts = tuner.sweep(kernel, precision(tag), sizes, cands, reps=20, passes=3)
with open(out, "w", newline="") as fh:
    tuner.write_sweep_csv(pts, fh)
best = {}
for p in pts:
    b = best.get(p.size)
    if b is None or p.measured_gbs > b.measured_gbs:
        best[p.size] = p
for n in sizes:
    base = next(p for p in pts if p.size == n and p.config.is_auto)
    print(n, f"auto {base.measured_gbs:.0f}", f"best {best[n].config.label()} {best[n].measured_gbs:.0f} "
          f"({best[n].measured_gbs / base.measured_gbs:.3f})", flush=True)
