#!/usr/bin/env python
"""Does the streaming rate depend on WHERE the operand sits in HBM?  Times
one op/size with the operand allocated behind a spacer of each given size
(MiB), through the plain entry point of the in-tree library.

    python scripts/alloc_offset_probe.py ssymv 32768 0,2,4,8,64,1024
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import OPS, alg_bytes  # noqa: E402
from paper_1410_1726_b200 import _lib  # noqa: E402
from paper_1410_1726_b200.core import precision  # noqa: E402

opname, n = sys.argv[1], int(sys.argv[2])
spacers = [int(s) for s in sys.argv[3].split(",")]
lib = _lib.load()
tag, family, op, herm = OPS[opname]
p = precision(tag)
name = {("s", False): "ssymv", ("d", False): "dsymv", ("c", True): "chemv", ("z", True): "zhemv"}[(tag, herm)]
fn = getattr(lib, f"kblas_{name}_async")
st = torch.cuda.current_stream().cuda_stream
one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)
nbytes = alg_bytes(tag, family, n, n, op)
for sp in spacers:
    spacer = torch.empty(max(1, sp << 20), dtype=torch.uint8, device="cuda")
    A = torch.empty(n, n, dtype=p.torch_dtype, device="cuda")
    (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1)
    x = torch.ones(n, dtype=p.torch_dtype, device="cuda")
    y = torch.empty(n, dtype=p.torch_dtype, device="cuda")
    call = lambda: fn(op.encode(), n, one, A.data_ptr(), n, x.data_ptr(), 1, zero, y.data_ptr(), 1, st)
    for _ in range(3):
        call()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            call()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 10)
    print(json.dumps({"op": opname, "n": n, "spacer_mib": sp, "A_addr_mib": (A.data_ptr() >> 20),
                      "A_addr_mod_2m": A.data_ptr() % (2 << 20), "gbs": round(nbytes / (best * 1e-3) / 1e9, 1),
                      "plan": _lib.last_plan()}), flush=True)
    del A, x, y, spacer
    torch.cuda.empty_cache()
