#!/usr/bin/env python
"""Small-N probe: a few calls of each op at N <= 8192, for an ncu launch
list (per-kernel device time of the streaming kernel vs its epilogue).

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/small.csv python scripts/small_n_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import OPS  # noqa: E402
from paper_1410_1726_b200 import _lib  # noqa: E402
from paper_1410_1726_b200.core import precision  # noqa: E402

ops = (sys.argv[1] if len(sys.argv) > 1 else "dgemv,dgemv_t,zgemv,sgemv,dsymv,zhemv,ssymv").split(",")
sizes = [int(s) for s in (sys.argv[2] if len(sys.argv) > 2 else "1024,2048,4096,8192").split(",")]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
lib = _lib.load()
sh = torch.cuda.current_stream().cuda_stream
for opname in ops:
    tag, family, op, herm = OPS[opname]
    p = precision(tag)
    one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)
    for n in sizes:
        # rotate over copies (> 512 MB together) so A streams from HBM even
        # when ncu runs with --cache-control none
        ncop = max(1, min(64, (512 << 20) // (n * n * p.element_bytes)))
        As = [torch.rand(n, n, dtype=p.torch_dtype, device="cuda") for _ in range(ncop)]
        x = torch.rand(n, dtype=p.torch_dtype, device="cuda")
        y = torch.rand(n, dtype=p.torch_dtype, device="cuda")
        for k in range(reps):
            A = As[k % ncop]
            if family == "symv":
                name = {("s", False): "ssymv", ("d", False): "dsymv", ("c", True): "chemv", ("z", True): "zhemv"}[(tag, herm)]
                rc = getattr(lib, f"kblas_{name}_async")(op.encode(), n, one, A.data_ptr(), n, x.data_ptr(), 1, zero,
                                                       y.data_ptr(), 1, sh)
            else:
                rc = getattr(lib, f"kblas_{tag}gemv_async")(op.encode(), n, n, one, A.data_ptr(), n, x.data_ptr(), 1,
                                                          zero, y.data_ptr(), 1, sh)
            assert rc == 0
        torch.cuda.synchronize()
        print(opname, n, _lib.last_plan(), flush=True)
