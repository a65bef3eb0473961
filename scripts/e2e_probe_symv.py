#!/usr/bin/env python
"""Per-call wall times of the numpy-vector DSYMV call at BASELINE
configs[1] (N=32768, A resident), to separate steady state from outliers.

    python scripts/e2e_probe_symv.py [n] [calls]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1410_1726_b200 as kb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 40
A = torch.empty(n, n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
hv = kb.HermitianView(kb.view_of(A.T), "l")
hx = torch.empty(n, dtype=torch.float64, pin_memory=True).uniform_(-1, 1)
hy = torch.empty(n, dtype=torch.float64, pin_memory=True)
npx, npy = hx.numpy(), hy.numpy()
ts = []
for i in range(calls):
    t0 = time.perf_counter()
    out = kb.symv_hemv("l", 1.0, hv, npx, 0.0, npy).y_out
    ts.append((time.perf_counter() - t0) * 1e3)
nbytes = 8 * (n * (n + 1) // 2 + 3 * n)
print("per-call ms:", " ".join(f"{t:.3f}" for t in ts))
st = sorted(ts[2:])
print(f"median {st[len(st) // 2]:.3f} ms = {nbytes / st[len(st) // 2] / 1e6:.0f} GB/s; min {st[0]:.3f}; max {st[-1]:.3f}")
