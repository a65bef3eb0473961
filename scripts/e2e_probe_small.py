#!/usr/bin/env python
"""Where a small numpy-vector call (BASELINE configs[0], DGEMV-N 4096)
loses time against its device-timed step: wall time per call of each layer
of the host path, A HBM-resident (4 rotating copies, > L2).

    python scripts/e2e_probe_small.py [n] [op]
"""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1410_1726_b200 as kb  # noqa: E402
from paper_1410_1726_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
NC = 4
As = [torch.empty(n, n, dtype=torch.float64, device="cuda").uniform_(-1, 1) for _ in range(NC)]
views = [kb.view_of(a.T) for a in As]
hx = torch.empty(n, dtype=torch.float64, pin_memory=True).uniform_(-1, 1)
hy = torch.empty(n, dtype=torch.float64, pin_memory=True)
npx, npy = hx.numpy(), hy.numpy()
xd = hx.cuda()
yd = torch.empty(n, dtype=torch.float64, device="cuda")
lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
one, zero = ctypes.c_double(1.0), ctypes.c_double(0.0)
cnt = [0]


def nxt():
    cnt[0] += 1
    return As[cnt[0] % NC]


def wall(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6


def dev_loop(reps=200):
    def call():
        lib.kblas_dgemv_async(b"n", n, n, 1.0, nxt().data_ptr(), n, xd.data_ptr(), 1, 0.0, yd.data_ptr(), 1, st)
    for _ in range(10):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def async_sync():
    lib.kblas_dgemv_async(b"n", n, n, 1.0, nxt().data_ptr(), n, xd.data_ptr(), 1, 0.0, yd.data_ptr(), 1, st)
    lib.kblas_stream_sync(st)


def c_hostvec():
    rc = lib.kblas_mv_hostvec(b"d", b"g", b"n", 0, n, n, ctypes.addressof(one), nxt().data_ptr(), n, 0, 0,
                              hx.data_ptr(), ctypes.addressof(zero), None, hy.data_ptr(), st)
    assert rc == 0


def api_numpy():
    cnt[0] += 1
    return kb.gemv("n", 1.0, views[cnt[0] % NC], npx, 0.0, npy).y_out


def api_torch_dev():
    cnt[0] += 1
    return kb.gemv("n", 1.0, views[cnt[0] % NC], xd, 0.0, yd).y_out


def h2d_kernel_d2h_torch():
    xd.copy_(hx, non_blocking=True)
    lib.kblas_dgemv_async(b"n", n, n, 1.0, nxt().data_ptr(), n, xd.data_ptr(), 1, 0.0, yd.data_ptr(), 1, st)
    hy.copy_(yd, non_blocking=True)
    torch.cuda.current_stream().synchronize()


rows = [("device-timed kernel loop (events)", dev_loop()),
        ("kblas_dgemv_async + kblas_stream_sync (device x, y)", wall(async_sync)),
        ("C kblas_mv_hostvec (pinned x, y)", wall(c_hostvec)),
        ("H2D + kblas_dgemv_async + D2H + sync (torch copies)", wall(h2d_kernel_d2h_torch)),
        ("kb.gemv torch device x, y", wall(api_torch_dev)),
        ("kb.gemv numpy x, y (pinned)", wall(api_numpy))]
nbytes = 8 * (n * n + 3 * n)
for name, us in rows:
    print(f"{name:56s} {us:8.2f} us  {nbytes / us / 1e3:8.0f} GB/s")
