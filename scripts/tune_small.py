#!/usr/bin/env python
"""Small/medium-N form choice: time each op per size with the library's
alternative forms forced on and off (GEMV-N split form, narrow SYMV tiles,
SSYMV TMA kernel), throughput over rotating operand copies as in
scripts/sweep.py.  One JSON line per (op, n, form).

    python scripts/tune_small.py [--ops ...] [--sizes ...] [--out FILE]
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

from bench import OPS, alg_bytes  # noqa: E402
from paper_1410_1726_b200 import _lib  # noqa: E402
from paper_1410_1726_b200.core import precision  # noqa: E402
from sweep import measure  # noqa: E402


def measure_graph(fn, reps, ncopies):
    """Device-side time per call: `calls` launches captured in one CUDA
    graph and replayed (no host launch overhead in the timed region)."""
    calls = max(reps, ncopies)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(0)  # the library's per-stream workspace is allocated outside the capture
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for k in range(calls):
                fn(k % ncopies)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / calls


def forms(family, op, tag):
    if family == "gemv" and op == "n":
        lib = _lib.load()
        f = {"auto": lambda: reset(), "stacked": lambda: _lib.set_gemv_split(0),
             "split_slots": lambda: (_lib.set_gemv_split(1), lib.kblas_set_gemv_cluster(0)),
             "split_cluster": lambda: (_lib.set_gemv_split(1), lib.kblas_set_gemv_cluster(1))}
        return f
    if family == "gemv":
        return {"auto": lambda: _lib.load().kblas_set_gemv_tc(-1, 80 << 20),
                "tc": lambda: _lib.load().kblas_set_gemv_tc(1, 0),
                "streamk": lambda: _lib.load().kblas_set_gemv_tc(0, 0)}
    if family == "gemv":
        return {"auto": lambda: _lib.load().kblas_set_gemv_tc(-1, 80 << 20),
                "tc": lambda: _lib.load().kblas_set_gemv_tc(1, 0),
                "streamk": lambda: _lib.load().kblas_set_gemv_tc(0, 0)}
    if family == "symv":
        big = 1 << 30
        lib = _lib.load()
        f = {"auto": lambda: reset(),
             "narrow": lambda: (_lib.set_symv_narrow(big), _lib.set_tma(0)),
             "mid": lambda: (_lib.set_symv_narrow(0), lib.kblas_set_symv_mid(big), _lib.set_tma(0)),
             "wide": lambda: (_lib.set_symv_narrow(0), lib.kblas_set_symv_mid(0), _lib.set_tma(0))}
        if tag == "s":
            f["tma"] = lambda: (_lib.set_symv_narrow(0), _lib.set_tma(1))
        return f
    return {"auto": lambda: None}


DEFAULTS = {}


def reset():
    _lib.set_gemv_split(-1)
    _lib.load().kblas_set_gemv_cluster(-1)
    _lib.load().kblas_set_gemv_split_waves(1)
    _lib.load().kblas_set_gemv_tc(-1, 80 << 20)
    _lib.set_tma(-1)
    if not DEFAULTS:  # the library's built-in thresholds
        DEFAULTS["narrow"] = _lib.set_symv_narrow(0)
        DEFAULTS["mid"] = _lib.load().kblas_set_symv_mid(0)
    _lib.set_symv_narrow(DEFAULTS["narrow"])
    _lib.load().kblas_set_symv_mid(DEFAULTS["mid"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", default="dgemv,sgemv,zgemv,cgemv,dgemv_t,zgemv_c,dsymv,zhemv,ssymv,chemv,dsymv_u")
    ap.add_argument("--sizes", default="1024,2048,3072,4096,6144,8192,12288,16384")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--out", default=None)
    ap.add_argument("--graph", action="store_true", help="also time calls replayed from a CUDA graph")
    args = ap.parse_args()
    lib = _lib.load()
    reset()
    out = open(args.out, "w") if args.out else None
    for opname in args.ops.split(","):
        tag, family, op, herm = OPS[opname]
        p = precision(tag)
        for n in [int(s) for s in args.sizes.split(",")]:
            ld = -(-n // 32) * 32
            mat = n * ld * p.element_bytes
            ncop = max(1, min(64, -(-(512 << 20) // mat)))
            As = []
            for _ in range(ncop):
                A = torch.empty(n, ld, dtype=p.torch_dtype, device="cuda")
                (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1)
                As.append(A)
            x = torch.empty(n, dtype=p.torch_dtype, device="cuda")
            (torch.view_as_real(x) if p.is_complex else x).uniform_(-1, 1)
            y = torch.empty(n, dtype=p.torch_dtype, device="cuda")
            one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)
            if family == "symv":
                name = {("s", False): "ssymv", ("d", False): "dsymv", ("c", True): "chemv",
                        ("z", True): "zhemv"}[(tag, herm)]
                f = getattr(lib, f"kblas_{name}_async")

                def call(k):
                    assert f(op.encode(), n, one, As[k].data_ptr(), ld, x.data_ptr(), 1, zero, y.data_ptr(), 1,
                             torch.cuda.current_stream().cuda_stream) == 0
            else:
                f = getattr(lib, f"kblas_{tag}gemv_async")

                def call(k):
                    assert f(op.encode(), n, n, one, As[k].data_ptr(), ld, x.data_ptr(), 1, zero, y.data_ptr(), 1,
                             torch.cuda.current_stream().cuda_stream) == 0
            nbytes = alg_bytes(tag, family, n, n, op)
            ref = None
            for form, setf in forms(family, op, tag).items():
                setf()
                ms = measure(call, args.reps, ncop)
                gms = measure_graph(call, args.reps, ncop) if args.graph else None
                call(0)
                torch.cuda.synchronize()
                got = y.clone()
                if ref is None:
                    ref = got
                diff = float(((got - ref).abs().max() / ref.abs().max()).item())
                row = {"op": opname, "n": n, "form": form, "us": round(ms * 1e3, 2),
                       "gbs": round(nbytes / ms / 1e6, 1),
                       "graph_us": round(gms * 1e3, 2) if gms else None,
                       "graph_gbs": round(nbytes / gms / 1e6, 1) if gms else None,
                       "plan": _lib.last_plan(), "rel_diff_vs_auto": diff}
                print(json.dumps(row), flush=True)
                if out:
                    out.write(json.dumps(row) + "\n")
                    out.flush()
            reset()
            del As
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
