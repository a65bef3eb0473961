#!/usr/bin/env python
"""Where the end-to-end (numpy x, y) call loses time against the
device-timed step at DSYMV N=32768: wall time per call for the public API
and for the raw C host-vector entry, next to the main kernel's event time.
"""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1410_1726_b200 as kb  # noqa: E402
from paper_1410_1726_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
A = torch.empty(n, n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
view = kb.view_of(A.T)
hv = kb.HermitianView(view, "l")
hx = torch.empty(n, dtype=torch.float64, pin_memory=True).uniform_(-1, 1)
hy = torch.empty(n, dtype=torch.float64, pin_memory=True)
npx, npy = hx.numpy(), hy.numpy()
xd = hx.cuda()
yd = torch.empty(n, dtype=torch.float64, device="cuda")
lib = _lib.load()
one, zero = ctypes.c_double(1.0), ctypes.c_double(0.0)
st = torch.cuda.current_stream().cuda_stream


def wall(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6


def dev_loop(reps=30):
    for _ in range(3):
        lib.kblas_dsymv_async(b"l", n, 1.0, A.data_ptr(), n, xd.data_ptr(), 1, 0.0, yd.data_ptr(), 1, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lib.kblas_dsymv_async(b"l", n, 1.0, A.data_ptr(), n, xd.data_ptr(), 1, 0.0, yd.data_ptr(), 1, st)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


_lib.timing_enable(True)
wall(lambda: lib.kblas_dsymv_async(b"l", n, 1.0, A.data_ptr(), n, xd.data_ptr(), 1, 0.0, yd.data_ptr(), 1, st))
_lib.timing_enable(False)
ms, cnt = _lib.timing_read()
print(f"n={n}")
print(f"main kernel (events)                 {ms / cnt * 1e3:8.1f} us")
print(f"device loop, back to back            {dev_loop():8.1f} us")
print(f"async call + sync each (device vecs) {wall(lambda: (lib.kblas_dsymv_async(b'l', n, 1.0, A.data_ptr(), n, xd.data_ptr(), 1, 0.0, yd.data_ptr(), 1, st), torch.cuda.synchronize())):8.1f} us")
print(f"C hostvec entry (pinned x, y)        {wall(lambda: lib.kblas_mv_hostvec(b'd', b's', b'l', 0, n, n, ctypes.addressof(one), A.data_ptr(), n, 0, 0, npx.ctypes.data, ctypes.addressof(zero), None, npy.ctypes.data, st)):8.1f} us")
print(f"kb.symv_hemv numpy x, y              {wall(lambda: kb.symv_hemv('l', 1.0, hv, npx, 0.0, npy)):8.1f} us")
print(f"kb.symv_hemv torch device x, y       {wall(lambda: (kb.symv_hemv('l', 1.0, hv, xd, 0.0, yd), torch.cuda.synchronize())):8.1f} us")
