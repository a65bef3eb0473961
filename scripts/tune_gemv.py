#!/usr/bin/env python
"""GEMV kernel-shape tuner: times every kblas_set_gemv_variant shape
against the default on the same HBM-resident operands (sizes >= 8k, so
every call streams from HBM) and checks the results agree.  JSON lines."""
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
    ap.add_argument("--ops", default="zgemv,zgemv_c,dgemv,dgemv_t,sgemv,sgemv_t,cgemv,cgemv_c")
    ap.add_argument("--sizes", default="16384,32768")
    ap.add_argument("--variants", default="0,3,4")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    lib = _lib.load()
    out = open(args.out, "w") if args.out else None
    sh = torch.cuda.current_stream().cuda_stream
    for opname in args.ops.split(","):
        tag, family, op, herm = OPS[opname]
        p = precision(tag)
        f = getattr(lib, f"kblas_{tag}gemv_async")
        one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)
        for n in [int(s) for s in args.sizes.split(",")]:
            # rotate over operand copies (> 512 MB together) so small sizes
            # stream from HBM rather than the 126 MB L2
            ncop = max(1, min(64, -(-(512 << 20) // (n * n * p.element_bytes))))
            As = []
            for _ in range(ncop):
                A = torch.empty(n, n, dtype=p.torch_dtype, device="cuda")
                (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1)
                As.append(A)
            x = torch.empty(n, dtype=p.torch_dtype, device="cuda")
            (torch.view_as_real(x) if p.is_complex else x).uniform_(-1, 1)
            y = torch.zeros(n, dtype=p.torch_dtype, device="cuda")

            ctr = [0]

            def call():
                A = As[ctr[0] % ncop]
                ctr[0] += 1
                assert f(op.encode(), n, n, one, A.data_ptr(), n, x.data_ptr(), 1, zero, y.data_ptr(), 1, sh) == 0

            nbytes = alg_bytes(tag, family, n, n, op)
            ref = None
            for v in [int(s) for s in args.variants.split(",")]:
                lib.kblas_set_gemv_variant(v)
                for _ in range(3):
                    call()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = max(args.reps, ncop)
                e0.record()
                for _ in range(reps):
                    call()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                ctr[0] = 0
                call()
                torch.cuda.synchronize()
                res = y.clone()
                if ref is None:
                    ref = res
                err = float((res - ref).abs().max() / (ref.abs().max() + 1e-30))
                row = {"op": opname, "n": n, "variant": v, "gbs": round(nbytes / ms / 1e6, 1),
                       "rel_diff_vs_default": err, "plan": _lib.last_plan()}
                print(json.dumps(row), flush=True)
                if out:
                    out.write(json.dumps(row) + "\n")
            lib.kblas_set_gemv_variant(0)
            del As
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
