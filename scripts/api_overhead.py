#!/usr/bin/env python
"""Host overhead of the public Python API (tiny operands, so the kernels
are negligible): per-call wall time of kb.symv_hemv / kb.gemv with device
operands and with numpy operands, vs the raw C-ABI call."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1410_1726_b200 as kb  # noqa: E402
from paper_1410_1726_b200 import _lib  # noqa: E402


def per_call(fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


d = 256
A = torch.rand(d, d, dtype=torch.float64, device="cuda")
v = kb.view_of(A.T)
hv = kb.HermitianView(v, "l")
x = torch.rand(d, dtype=torch.float64, device="cuda")
y = torch.rand(d, dtype=torch.float64, device="cuda")
hx = torch.rand(d, dtype=torch.float64).pin_memory().numpy()
hy = torch.rand(d, dtype=torch.float64).pin_memory().numpy()
lib = _lib.load()
one, zero = _lib.scalar("d", 1.0), _lib.scalar("d", 0.0)
sh = torch.cuda.current_stream().cuda_stream
print("raw C ABI dsymv_async      %.1f us" % per_call(
    lambda: lib.kblas_dsymv_async(b"l", d, one, A.data_ptr(), d, x.data_ptr(), 1, zero, y.data_ptr(), 1, sh)))
print("kb.symv_hemv torch in/out  %.1f us" % per_call(lambda: kb.symv_hemv("l", 1.0, hv, x, 0.0, y)))
print("kb.symv_hemv inplace       %.1f us" % per_call(lambda: kb.symv_hemv("l", 1.0, hv, x, 0.0, y, inplace=True)))
print("kb.symv_hemv numpy x,y     %.1f us" % per_call(lambda: kb.symv_hemv("l", 1.0, hv, hx, 0.0, hy), 500))
print("kb.gemv torch in/out       %.1f us" % per_call(lambda: kb.gemv("n", 1.0, v, x, 0.0, y)))

if len(sys.argv) > 1 and sys.argv[1] == "profile":
    import cProfile
    import pstats

    pr = cProfile.Profile()
    pr.enable()
    for _ in range(2000):
        kb.symv_hemv("l", 1.0, hv, hx, 0.0, hy)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
