#!/usr/bin/env python
"""Row-owning GEMV-N (kblas_set_gemv_split(3), configuration index via
kblas_set_gemv_rowown) against the default choice at small N: interleaved
best-of-3 windows over rotating operand copies (> 512 MB together)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch  # noqa: E402

from bench import alg_bytes  # noqa: E402
from paper_1410_1726_b200 import _lib  # noqa: E402
from paper_1410_1726_b200.core import precision  # noqa: E402
from sweep import measure  # noqa: E402

tags = (sys.argv[1] if len(sys.argv) > 1 else "d,z,c,s").split(",")
sizes = [int(s) for s in (sys.argv[2] if len(sys.argv) > 2 else "1024,2048,3072,4096,6144,8192").split(",")]
cfgs = [int(s) for s in (sys.argv[3] if len(sys.argv) > 3 else "0,1,2,3,4,5").split(",")]
lib = _lib.load()
sh = torch.cuda.current_stream().cuda_stream
for tag in tags:
    p = precision(tag)
    one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)
    for n in sizes:
        ncop = max(1, min(64, -(-(512 << 20) // (n * n * p.element_bytes))))
        As = []
        for _ in range(ncop):
            A = torch.empty(n, n, dtype=p.torch_dtype, device="cuda")
            (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1)
            As.append(A)
        x = torch.empty(n, dtype=p.torch_dtype, device="cuda")
        (torch.view_as_real(x) if p.is_complex else x).uniform_(-1, 1)
        y = torch.empty(n, dtype=p.torch_dtype, device="cuda")
        f = getattr(lib, f"kblas_{tag}gemv_async")

        def call(k):
            assert f(b"n", n, n, one, As[k].data_ptr(), n, x.data_ptr(), 1, zero, y.data_ptr(), 1, sh) == 0

        arms = [("default", None)] + [(f"ro{c}", c) for c in cfgs]
        best, plans, ys = {}, {}, {}
        for _ in range(3):
            for name, c in arms:
                prev = lib.kblas_set_gemv_split(3 if c is not None else -1)
                prev_c = lib.kblas_set_gemv_rowown(c if c is not None else -1)
                t = measure(call, 20, ncop)
                call(0)
                torch.cuda.synchronize()
                plans[name], ys[name] = _lib.last_plan(), y.clone()
                lib.kblas_set_gemv_split(prev)
                lib.kblas_set_gemv_rowown(prev_c)
                best[name] = min(best.get(name, 1e9), t)
        nb = alg_bytes(tag, "gemv", n, n, "n")
        ref = ys["default"]
        for name, _ in arms:
            d = float((ys[name] - ref).abs().max()) / (float(ref.abs().max()) or 1.0)
            print(json.dumps({"prec": tag, "n": n, "arm": name, "gbs": round(nb / best[name] / 1e6, 1),
                              "rel_diff": d, "plan": plans[name]}), flush=True)
        del As
        torch.cuda.empty_cache()
