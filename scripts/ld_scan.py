#!/usr/bin/env python
"""Sensitivity of the streaming kernels to the leading dimension: the same
N with ld = N and padded ld values (DRAM channel aliasing of power-of-two
column strides).  One JSON line per (op, n, ld)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import OPS, alg_bytes  # noqa: E402
from paper_1410_1726_b200 import _lib  # noqa: E402
from paper_1410_1726_b200.core import precision  # noqa: E402

ops = (sys.argv[1] if len(sys.argv) > 1 else "dsymv,dgemv_t,dgemv").split(",")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
pads = [int(s) for s in (sys.argv[3] if len(sys.argv) > 3 else "0,32,64,128,256,512,1024,4096").split(",")]
lib = _lib.load()
sh = torch.cuda.current_stream().cuda_stream
for opname in ops:
    tag, family, op, herm = OPS[opname]
    p = precision(tag)
    one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)
    for pad in pads:
        ld = n + pad
        A = torch.empty(n, ld, dtype=p.torch_dtype, device="cuda")
        (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1)
        x = torch.empty(n, dtype=p.torch_dtype, device="cuda")
        (torch.view_as_real(x) if p.is_complex else x).uniform_(-1, 1)
        y = torch.empty(n, dtype=p.torch_dtype, device="cuda")
        if family == "symv":
            name = {("s", False): "ssymv", ("d", False): "dsymv", ("c", True): "chemv", ("z", True): "zhemv"}[(tag, herm)]
            f = getattr(lib, f"kblas_{name}_async")

            def call():
                assert f(op.encode(), n, one, A.data_ptr(), ld, x.data_ptr(), 1, zero, y.data_ptr(), 1, sh) == 0
        else:
            f = getattr(lib, f"kblas_{tag}gemv_async")

            def call():
                assert f(op.encode(), n, n, one, A.data_ptr(), ld, x.data_ptr(), 1, zero, y.data_ptr(), 1, sh) == 0
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 30
        e0.record()
        for _ in range(reps):
            call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        nbytes = alg_bytes(tag, family, n, n, op)
        print(json.dumps({"op": opname, "n": n, "ld": ld, "gbs": round(nbytes / ms / 1e6, 1)}), flush=True)
        del A
        torch.cuda.empty_cache()
