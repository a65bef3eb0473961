"""Per-piece Python cost of the numpy-vector call path (GPU box):
each helper timed alone over many iterations."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1410_1726_b200 as kb
from paper_1410_1726_b200 import _ops, _lib, kernels, roofline

n = 4096
A = torch.empty(n, n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
v = kb.view_of(A.T)
x = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy(); x[:] = 1
y = np.zeros(n)
dev = _ops.device_for(v, y, x)
prec = v.precision

def t(name, fn, k=20000):
    for _ in range(200): fn()
    t0 = time.perf_counter()
    for _ in range(k): fn()
    print(f"{name:40s} {(time.perf_counter() - t0) / k * 1e6:7.3f} us")

t("device_for", lambda: _ops.device_for(v, y, x))
t("host_vectors", lambda: _ops.host_vectors(x, y, False))
t("_is_zero(alpha)", lambda: kernels._is_zero(1.0))
t("matrix_in", lambda: _ops.matrix_in(v, dev))
t("_PINNED.get", lambda: _ops._PINNED.get(n, torch.float64))
def ondev():
    with _ops._on_device(dev):
        pass
t("_on_device", ondev)
t("stream_handle", lambda: _ops.stream_handle(dev))
t("_HC.last_plan", lambda: _ops._HC.last_plan())
t("DeferredReport", lambda: kernels._DeferredReport(y, lambda: None))
out, out_np = _ops._PINNED.get(n, torch.float64)
sh = _ops.stream_handle(dev)
ptr, lda, keep = _ops.matrix_in(v, dev)
t("_HC.mv_hostvec sync (C+GPU)", lambda: _ops._HC.mv_hostvec("d", "g", "n", 0, n, n, 1.0, ptr, lda, 0, 0, x, n, 0.0, y, n, out.data_ptr(), sh, True), 2000)
t("kb.gemv numpy sync", lambda: kb.gemv("n", 1.0, v, x, 0.0, y), 2000)
t("trans.lower + checks", lambda: ("n".lower() in ("n", "t", "c"), isinstance(v, kb.MatrixView)))
t("out.data_ptr()", lambda: out.data_ptr())
