#!/usr/bin/env python
"""Host (CPU) cost per call of the numpy-vector path, sync and queued, at a
tiny order (n=256, the kernels take a few microseconds) and at BASELINE
configs[0] (DGEMV-N 4096), plus a cProfile of the queued loop.

    python scripts/queue_overhead.py [n]
"""
import ctypes
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1410_1726_b200 as kb  # noqa: E402
from paper_1410_1726_b200 import _lib  # noqa: E402

lib = _lib.load()


def setup(n, nc):
    As = [torch.empty(n, n, dtype=torch.float64, device="cuda").uniform_(-1, 1) for _ in range(nc)]
    views = [kb.view_of(a.T) for a in As]
    hxs = [torch.empty(n, dtype=torch.float64, pin_memory=True).uniform_(-1, 1) for _ in range(16)]
    return As, views, hxs


def per_call(fn, reps):
    for i in range(20):
        fn(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(reps):
        fn(i)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6


for n, nc in ((256, 1), (4096, 4)):
    As, views, hxs = setup(n, nc)
    npxs = [h.numpy() for h in hxs]
    hy = torch.empty(n, dtype=torch.float64, pin_memory=True)
    npy = hy.numpy()
    st = torch.cuda.current_stream().cuda_stream
    one, zero = ctypes.c_double(1.0), ctypes.c_double(0.0)
    xd = hxs[0].cuda()
    yd = torch.empty(n, dtype=torch.float64, device="cuda")

    def dev_async(i):
        lib.kblas_dgemv_async(b"n", n, n, 1.0, As[i % nc].data_ptr(), n, xd.data_ptr(), 1, 0.0, yd.data_ptr(), 1, st)

    def c_hostvec_async(i):
        lib.kblas_mv_hostvec_async(b"d", b"g", b"n", 0, n, n, ctypes.addressof(one), As[i % nc].data_ptr(), n, 0, 0,
                                   hxs[i % 16].data_ptr(), ctypes.addressof(zero), None, hy.data_ptr(), st)

    def api_sync(i):
        return kb.gemv("n", 1.0, views[i % nc], npxs[i % 16], 0.0, npy).y_out

    q = kb.CommandQueue()
    hs = []

    def api_queued(i):
        hs.append(kb.gemv_async("n", 1.0, views[i % nc], npxs[i % 16], 0.0, npy, queue=q))
        if len(hs) == 16:
            q.synchronize()
            for h in hs:
                float(h.result().y_out[0])
            hs.clear()

    print(f"n={n}")
    for name, fn in (("ctypes kblas_dgemv_async (device x,y)", dev_async),
                     ("ctypes kblas_mv_hostvec_async (pinned)", c_hostvec_async),
                     ("kb.gemv numpy (sync)", api_sync),
                     ("kb.gemv_async numpy (queue, sync/16)", api_queued)):
        print(f"  {name:44s} {per_call(fn, 2000 if n == 256 else 500):8.2f} us/call")
    if n == 256:
        pr = cProfile.Profile()
        pr.enable()
        for i in range(2000):
            api_queued(i)
        torch.cuda.synchronize()
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(22)
