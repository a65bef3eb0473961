#!/usr/bin/env python
"""BASELINE configs[3]: GEMV / SYMV on a misaligned submatrix through the
offset API (reference offset.py:83-208).

Parent: 16384 x 16384 (ld 16384) in HBM.  For each offset (i, j) the
submatrix is parent[i:, j:] (SYMV: the diagonal block at (i, i)).  Ours:
kblas_xgemv_offset / kblas_xsymv_offset with the parent pointer and the
offsets.  Comparator: cuBLAS on the shifted pointer (the "standard kernel on
a misaligned view" of the paper).  GB/s counts only the true submatrix.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import torch  # noqa: E402

from paper_1410_1726_b200 import _lib, roofline  # noqa: E402
from paper_1410_1726_b200.core import precision  # noqa: E402
from sweep import Cublas  # noqa: E402


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--tags", default="d,s,z,c")
    ap.add_argument("--offsets", default="0:0,1:1,7:3,13:13,16:16,3:0,5:0,31:0,33:0")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    lib = _lib.load()
    cub = Cublas()
    dev = torch.device("cuda", 0)
    out = open(args.out, "w") if args.out else None
    N = args.n
    for tag in args.tags.split(","):
        p = precision(tag)
        A = torch.empty(N, N, dtype=p.torch_dtype, device=dev)
        (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1)
        x = torch.empty(N, dtype=p.torch_dtype, device=dev)
        (torch.view_as_real(x) if p.is_complex else x).uniform_(-1, 1)
        y = torch.zeros(N, dtype=p.torch_dtype, device=dev)
        y2 = torch.zeros(N, dtype=p.torch_dtype, device=dev)
        sh = torch.cuda.current_stream().cuda_stream
        one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)
        es = p.element_bytes
        base = A.data_ptr()
        sname = {"s": "ssymv", "d": "dsymv", "c": "chemv", "z": "zhemv"}[tag]
        for spec in args.offsets.split(","):
            i, j = (int(v) for v in spec.split(":"))
            for op in ("gemv_n", "gemv_t", "symv_l"):
                if op == "symv_l" and i != j:
                    continue
                if op.startswith("gemv"):
                    tr = op[-1]
                    m, n = N - i, N - j
                    f = getattr(lib, f"kblas_{tag}gemv_offset_async")

                    def ours():
                        assert f(tr.encode(), m, n, one, base, N, x.data_ptr(), 1, zero, y.data_ptr(), 1, i, j, sh) == 0

                    def theirs():
                        cub.call(tag, "gemv", tr, False, m, n, base + (j * N + i) * es, N, x.data_ptr(), y2.data_ptr(), sh)

                    nbytes = roofline.gemv_bytes(p, m, n, tr)
                else:
                    d = N - i
                    f = getattr(lib, f"kblas_{sname}_offset_async")

                    def ours():
                        assert f(b"l", d, one, base, N, x.data_ptr(), 1, zero, y.data_ptr(), 1, i, sh) == 0

                    def theirs():
                        cub.call(tag, "symv", "l", tag in "cz", d, d, base + (i * N + i) * es, N, x.data_ptr(),
                                 y2.data_ptr(), sh)

                    nbytes = roofline.symv_bytes(p, d)
                ms = timeit(ours, args.reps)
                row = {"tag": tag, "op": op, "row_off": i, "col_off": j, "gbs": round(nbytes / ms / 1e6, 1),
                       "plan": _lib.last_plan()}
                if cub.lib is not None:
                    cms = timeit(theirs, args.reps)
                    row["cublas_gbs"] = round(nbytes / cms / 1e6, 1)
                    scale = float(y2.abs().max().item()) or 1.0
                    row["rel_diff_vs_cublas"] = float((y - y2).abs().max().item() / scale)
                print(json.dumps(row), flush=True)
                if out:
                    out.write(json.dumps(row) + "\n")
        del A
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
