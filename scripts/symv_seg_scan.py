#!/usr/bin/env python
"""SYMV/HEMV work schedule scan: contiguous stream-K against segments of K
items dealt round robin (kblas_set_symv_segment), same operands, same box.

For each op and order: whole-call time (main kernel + epilogue, best of
interleaved >= 2 ms windows) and the main kernel alone (the library's
event brackets), per K, plus the max relative difference of y against the
contiguous schedule (the t2 partials are summed in a different grouping).
Prints JSON lines.

    python scripts/symv_seg_scan.py --ops dsymv,zhemv --sizes 16384,32768 --ks 0,2,4,8
"""

from __future__ import annotations

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


def window(call, dev, min_ms=2.0):
    reps = 1
    while True:
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            call()
        e1.record()
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1)
        if ms >= min_ms or reps >= 4096:
            return ms / reps
        reps = max(reps * 2, int(reps * min_ms / max(ms, 1e-3)) + 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", default="dsymv,zhemv,ssymv,chemv")
    ap.add_argument("--sizes", default="16384,32768,40960")
    ap.add_argument("--ks", default="0,4")
    ap.add_argument("--windows", default="1", help="kblas_set_symv_window values (combined with every K)")
    ap.add_argument("--passes", type=int, default=3)
    ap.add_argument("--ldpad", type=int, default=0)
    args = ap.parse_args()
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    ks = [(int(k), int(b)) for k in args.ks.split(",") for b in args.windows.split(",")]
    for opname in args.ops.split(","):
        tag, family, op, herm = OPS[opname]
        p = precision(tag)
        name = {("s", False): "ssymv", ("d", False): "dsymv", ("c", True): "chemv", ("z", True): "zhemv"}[(tag, herm)]
        f = getattr(lib, f"kblas_{name}_async")
        for n in [int(s) for s in args.sizes.split(",")]:
            ld = n + args.ldpad
            A = torch.empty(n, ld, dtype=p.torch_dtype, device=dev)
            (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1)
            x = torch.empty(n, dtype=p.torch_dtype, device=dev)
            (torch.view_as_real(x) if p.is_complex else x).uniform_(-1, 1)
            ys = {k: torch.zeros(n, dtype=p.torch_dtype, device=dev) for k in ks}
            sh = torch.cuda.current_stream().cuda_stream
            one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)
            nbytes = alg_bytes(tag, family, n, n, op)

            def call_k(k):
                def call():
                    prev = lib.kblas_set_symv_segment(k[0])
                    prevw = lib.kblas_set_symv_window(k[1])
                    rc = f(op.encode(), n, one, A.data_ptr(), ld, x.data_ptr(), 1, zero, ys[k].data_ptr(), 1, sh)
                    lib.kblas_set_symv_segment(prev)
                    lib.kblas_set_symv_window(prevw)
                    assert rc == 0
                return call

            best = {k: 1e9 for k in ks}
            plans = {}
            for k in ks:  # warm: tile tables, workspace
                call_k(k)()
                torch.cuda.synchronize(dev)
                plans[k] = _lib.last_plan()
            for _ in range(args.passes):
                for k in ks:
                    best[k] = min(best[k], window(call_k(k), dev))
            kern = {}
            for k in ks:
                _lib.timing_read()
                _lib.timing_enable(True)
                for _ in range(10):
                    call_k(k)()
                torch.cuda.synchronize(dev)
                _lib.timing_enable(False)
                ms, cnt = _lib.timing_read()
                kern[k] = ms / max(cnt, 1)
            ref = ys[ks[0]]
            scale = float(ref.abs().max())
            for k in ks:
                print(json.dumps({
                    "op": opname, "n": n, "ld": ld, "K": k[0], "B": k[1], "ms": round(best[k], 5),
                    "gbs": round(nbytes / (best[k] * 1e-3) / 1e9, 1),
                    "kernel_ms": round(kern[k], 5), "kernel_gbs": round(nbytes / (kern[k] * 1e-3) / 1e9, 1),
                    "rel_diff_vs_first": float((ys[k] - ref).abs().max()) / scale, "plan": plans[k]}), flush=True)
            del A
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
