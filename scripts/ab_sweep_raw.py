#!/usr/bin/env python
"""Throughput of the plain BLAS-style entry points of one library build,
loaded straight with ctypes (no package import), so builds from other
commits with a different extended ABI can be timed on the same box.

    python scripts/ab_sweep_raw.py LIB.so OPS SIZES TAG

One JSON line per (op, n): GB/s on algorithmic bytes over >= 2 ms
windows of back-to-back calls, rotating over >= 512 MB of operand copies.
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import OPS, alg_bytes  # noqa: E402

DT = {"s": (torch.float32, 4), "d": (torch.float64, 8), "c": (torch.complex64, 8), "z": (torch.complex128, 16)}


class _C2f(ctypes.Structure):
    _fields_ = [("re", ctypes.c_float), ("im", ctypes.c_float)]


class _C2d(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


SCALAR = {"s": ctypes.c_float, "d": ctypes.c_double, "c": _C2f, "z": _C2d}


def scalar(tag, v):
    return SCALAR[tag](v) if tag in "sd" else SCALAR[tag](v, 0.0)


def main():
    lib = ctypes.CDLL(sys.argv[1])
    ops, sizes, tag_out = sys.argv[2].split(","), [int(s) for s in sys.argv[3].split(",")], sys.argv[4]
    st = torch.cuda.current_stream().cuda_stream
    for opname in ops:
        tag, family, op, herm = OPS[opname]
        dt, eb = DT[tag]
        if family == "symv":
            name = {("s", False): "ssymv", ("d", False): "dsymv", ("c", True): "chemv", ("z", True): "zhemv"}[(tag, herm)]
            fn = getattr(lib, f"kblas_{name}_async")
        else:
            fn = getattr(lib, f"kblas_{tag}gemv_async")
        fn.restype = ctypes.c_int
        S, P, I = SCALAR[tag], ctypes.c_void_p, ctypes.c_int
        dims = [I] if family == "symv" else [I, I]
        fn.argtypes = [ctypes.c_char] + dims + [S, P, I, P, I, S, P, I, P]
        for n in sizes:
            ld = -(-n // 32) * 32
            nc = max(1, min(64, -(-(1 << 30) // (n * ld * eb))))
            As = []
            for _ in range(nc):
                A = torch.empty(n, ld, dtype=dt, device="cuda")
                (torch.view_as_real(A) if tag in "cz" else A).uniform_(-1, 1)
                As.append(A)
            x = torch.ones(n, dtype=dt, device="cuda")
            y = torch.zeros(n, dtype=dt, device="cuda")
            one, zero = scalar(tag, 1.0), scalar(tag, 0.0)

            def call(i):
                a = As[i % nc].data_ptr()
                dims = (n,) if family == "symv" else (n, n)
                rc = fn(op.encode(), *dims, one, a, ld, x.data_ptr(), 1, zero, y.data_ptr(), 1, st)
                assert rc == 0, rc

            for i in range(3 * nc):
                call(i)
            torch.cuda.synchronize()
            best = float("inf")
            for _ in range(3):
                reps = 1
                while True:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for i in range(reps):
                        call(i)
                    e1.record()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1)
                    if ms >= 2.0:
                        break
                    reps *= 2
                best = min(best, ms / reps)
            nbytes = alg_bytes(tag, family, n, n, op)
            print(json.dumps({"lib": tag_out, "op": opname, "n": n, "gbs": round(nbytes / (best * 1e-3) / 1e9, 1)}),
                  flush=True)
            del As
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
