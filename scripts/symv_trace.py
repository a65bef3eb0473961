#!/usr/bin/env python
"""Per-CTA start / end times of the register SYMV/HEMV kernel
(kblas_set_symv_trace): how long the first CTAs to finish sit idle while
the last ones stream.  Prints JSON lines.  Needs an investigation build:
KBLAS_NVCC_EXTRA=-DKBLAS_SYMV_TRACE=1 python -m paper_1410_1726_b200._build --force

    python scripts/symv_trace.py [--ops dsymv,zhemv] [--sizes 32768,100000]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import OPS, alg_bytes  # noqa: E402
from paper_1410_1726_b200 import _lib  # noqa: E402
from paper_1410_1726_b200.core import precision  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ops", default="dsymv,zhemv,ssymv")
ap.add_argument("--sizes", default="16384,32768,65536,100000")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--per-cta", default=None, help="also write each run's per-CTA end times and SM ids here (JSON)")
args = ap.parse_args()
lib = _lib.load()
dev = torch.device("cuda", 0)
rows = []
trace = torch.zeros(3 * 4096, dtype=torch.int64, device=dev)
for opname in args.ops.split(","):
    tag, family, op, herm = OPS[opname]
    p = precision(tag)
    name = {("s", False): "ssymv", ("d", False): "dsymv", ("c", True): "chemv", ("z", True): "zhemv"}[(tag, herm)]
    fn = getattr(lib, f"kblas_{name}_async")
    for n in [int(s) for s in args.sizes.split(",")]:
        if n * n * p.element_bytes > torch.cuda.mem_get_info()[0] - (4 << 30):
            continue
        A = torch.empty(n, n, dtype=p.torch_dtype, device=dev)
        (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1)
        x = torch.ones(n, dtype=p.torch_dtype, device=dev)
        y = torch.empty(n, dtype=p.torch_dtype, device=dev)
        one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)
        st = torch.cuda.current_stream().cuda_stream
        call = lambda: fn(op.encode(), n, one, A.data_ptr(), n, x.data_ptr(), 1, zero, y.data_ptr(), 1, st)
        call()
        P = int(_lib.last_plan().split(" P=")[1].split()[0])
        res = []
        for r in range(args.reps):
            trace.zero_()
            if lib.kblas_set_symv_trace(trace.data_ptr()) != 0:
                sys.exit("this library was built without the trace: rebuild with "
                         "KBLAS_NVCC_EXTRA=-DKBLAS_SYMV_TRACE=1 python -m paper_1410_1726_b200._build --force")
            call()
            lib.kblas_set_symv_trace(None)
            torch.cuda.synchronize()
            t = trace[: 3 * P].view(P, 3).cpu()
            start, end, sm = t[:, 0], t[:, 1], t[:, 2]
            if args.per_cta:
                rows.append({"op": opname, "n": n, "rep": r, "end_us": ((end - start.min()).double() / 1e3).tolist(),
                             "sm": sm.tolist()})
            span = float(end.max() - start.min()) / 1e3
            idle = float((end.max() - end).double().mean()) / 1e3
            res.append((span, float(end.max() - end.min()) / 1e3, idle, float(start.max() - start.min()) / 1e3))
        best = min(res)
        print(json.dumps({"op": opname, "n": n, "ctas": P, "span_us": round(best[0], 1),
                          "finish_spread_us": round(best[1], 1), "mean_idle_us": round(best[2], 1),
                          "idle_frac": round(best[2] / best[0], 4), "start_spread_us": round(best[3], 1),
                          "plan": _lib.last_plan()}), flush=True)
        del A
        torch.cuda.empty_cache()
if args.per_cta:
    json.dump(rows, open(args.per_cta, "w"))
