#!/usr/bin/env python
"""Empirical tuner for the SYMV/HEMV streaming kernel (SURVEY §8f rank 1,
the B200 replacement of the reference's analytic tuner, tuner.py:168-222).

For each op and size, times the register-load kernel and every TMA
variant (kblas_set_symv_variant) on the same HBM-resident operands and
checks each result against the register kernel's.  Prints JSON lines.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", default="dsymv,zhemv,ssymv,chemv")
    ap.add_argument("--sizes", default="8192,16384,32768")
    ap.add_argument("--variants", default="0,1,103,105")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    out = open(args.out, "w") if args.out else None
    for opname in args.ops.split(","):
        tag, family, op, herm = OPS[opname]
        p = precision(tag)
        name = {("s", False): "ssymv", ("d", False): "dsymv", ("c", True): "chemv", ("z", True): "zhemv"}[(tag, herm)]
        f = getattr(lib, f"kblas_{name}_async")
        for n in [int(s) for s in args.sizes.split(",")]:
            A = torch.empty(n, n, dtype=p.torch_dtype, device=dev)
            (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1)
            x = torch.empty(n, dtype=p.torch_dtype, device=dev)
            (torch.view_as_real(x) if p.is_complex else x).uniform_(-1, 1)
            y = torch.zeros(n, dtype=p.torch_dtype, device=dev)
            sh = torch.cuda.current_stream().cuda_stream
            one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)

            def call():
                assert f(op.encode(), n, one, A.data_ptr(), n, x.data_ptr(), 1, zero, y.data_ptr(), 1, sh) == 0

            nbytes = alg_bytes(tag, family, n, n, op)
            ref = None
            for v in ["regs"] + args.variants.split(","):
                if v == "regs":
                    _lib.set_tma(False)
                    lib.kblas_set_symv_variant(-1)
                elif int(v) >= 100:
                    _lib.set_tma(False)
                    lib.kblas_set_symv_variant(int(v))
                else:
                    _lib.set_tma(True)
                    lib.kblas_set_symv_variant(int(v))
                for _ in range(3):
                    call()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(args.reps):
                    call()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / args.reps
                res = y.clone()
                if ref is None:
                    ref = res
                err = float((res - ref).abs().max() / (ref.abs().max() + 1e-30))
                row = {"op": opname, "n": n, "variant": v, "gbs": round(nbytes / ms / 1e6, 1), "ms": round(ms, 5),
                       "rel_diff_vs_regs": err, "plan": _lib.last_plan()}
                print(json.dumps(row), flush=True)
                if out:
                    out.write(json.dumps(row) + "\n")
            _lib.set_tma(-1)
            lib.kblas_set_symv_variant(-1)
            del A
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
