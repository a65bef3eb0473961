#!/usr/bin/env python
"""GEMV-N at small N, ours vs cuBLAS on the same buffers: a few calls of
each for an ncu launch list (grid, block, device time, DRAM bytes).

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size,launch__block_size \
        --clock-control none --csv --log-file gpurun_out/gemvn_small.csv python scripts/gemv_n_small_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch  # noqa: E402

from paper_1410_1726_b200 import _lib  # noqa: E402
from paper_1410_1726_b200.core import precision  # noqa: E402
from sweep import Cublas  # noqa: E402

ops = (sys.argv[1] if len(sys.argv) > 1 else "d,z,c").split(",")
sizes = [int(s) for s in (sys.argv[2] if len(sys.argv) > 2 else "2048,4096").split(",")]
lib = _lib.load()
cub = Cublas()
sh = torch.cuda.current_stream().cuda_stream
for tag in ops:
    p = precision(tag)
    one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)
    for n in sizes:
        ncop = max(1, min(16, -(-(512 << 20) // (n * n * p.element_bytes))))
        As = [torch.empty(n, n, dtype=p.torch_dtype, device="cuda") for _ in range(ncop)]
        for A in As:
            (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1)
        x = torch.ones(n, dtype=p.torch_dtype, device="cuda")
        y = torch.empty(n, dtype=p.torch_dtype, device="cuda")
        f = getattr(lib, f"kblas_{tag}gemv_async")
        for k in range(4):
            assert f(b"n", n, n, one, As[k % ncop].data_ptr(), n, x.data_ptr(), 1, zero, y.data_ptr(), 1, sh) == 0
        print(tag, n, _lib.last_plan(), flush=True)
        for k in range(4):
            cub.call(tag, "gemv", "n", False, n, n, As[k % ncop].data_ptr(), n, x.data_ptr(), y.data_ptr(), sh)
        torch.cuda.synchronize()
        del As
        torch.cuda.empty_cache()
