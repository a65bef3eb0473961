#!/usr/bin/env python
"""Size sweep (BASELINE configs[2] / [3]): achieved GB/s of every op and
precision vs N on one B200, with cuBLAS (libcublas from the torch wheel,
called through ctypes on the same buffers) as the library comparator.

    python scripts/sweep.py [--ops dsymv,zhemv,...] [--sizes 1024,...] [--out FILE]

Timing: CUDA events around back-to-back calls (throughput), best of
--passes windows interleaved with the cuBLAS (and --ab-table) arms.  Operands
smaller than 512 MB are replicated and the calls rotate over the copies,
so every call streams its matrix from HBM (the copies together exceed the
126 MB L2 by >4x).  `single_ms` is the median single-call time after a
512 MB L2 flush (latency, launch included).  GB/s uses the algorithmic
bytes (roofline.py / SURVEY §8d).
"""

from __future__ import annotations

import argparse
import ctypes
import glob
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import OPS, alg_bytes  # noqa: E402
from paper_1410_1726_b200 import _lib  # noqa: E402
from paper_1410_1726_b200.core import precision  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


class Cublas:
    def __init__(self):
        cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cublas", "lib",
                                       "libcublas.so*"))
        cands += ["libcublas.so.12", "/usr/local/cuda/lib64/libcublas.so"]
        self.lib = None
        for c in cands:
            try:
                self.lib = ctypes.CDLL(c)
                break
            except OSError:
                continue
        self.h = ctypes.c_void_p()
        if self.lib is None or self.lib.cublasCreate_v2(ctypes.byref(self.h)) != 0:
            self.lib = None

    def call(self, tag, family, op, herm, m, n, A, ld, x, y, stream):
        if self.lib is None:
            return False
        self.lib.cublasSetStream_v2(self.h, ctypes.c_void_p(stream))
        sc = {"s": ctypes.c_float, "d": ctypes.c_double}
        if tag in "sd":
            one, zero = sc[tag](1.0), sc[tag](0.0)
        else:
            t = ctypes.c_float if tag == "c" else ctypes.c_double
            one, zero = (t * 2)(1.0, 0.0), (t * 2)(0.0, 0.0)
        vp = ctypes.c_void_p
        if family == "symv":
            name = {"s": "Ssymv", "d": "Dsymv", "c": "Chemv" if herm else "Csymv", "z": "Zhemv" if herm else "Zsymv"}[tag]
            f = getattr(self.lib, f"cublas{name}_v2")
            uplo = 0 if op == "l" else 1  # CUBLAS_FILL_MODE_LOWER = 0
            rc = f(self.h, uplo, n, ctypes.byref(one), vp(A), ld, vp(x), 1, ctypes.byref(zero), vp(y), 1)
        else:
            f = getattr(self.lib, f"cublas{tag.upper()}gemv_v2")
            tr = {"n": 0, "t": 1, "c": 2}[op]
            rc = f(self.h, tr, m, n, ctypes.byref(one), vp(A), ld, vp(x), 1, ctypes.byref(zero), vp(y), 1)
        return rc == 0


def measure(fn, reps, ncopies, min_ms: float = 2.0):
    """Back-to-back calls (throughput); fn(k) uses operand copy k % ncopies so
    the operands streamed per window exceed the L2 several times over.  The
    window is at least `min_ms` long (more calls for small operands, whose
    single-call times are a few microseconds)."""
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k in range(3):
        fn(k % ncopies)
    torch.cuda.synchronize()
    e0.record()
    fn(0)
    e1.record()
    torch.cuda.synchronize()
    one = max(e0.elapsed_time(e1), 1e-3)
    calls = max(reps, ncopies, min(2000, int(min_ms / one) + 1))
    e0.record()
    for k in range(calls):
        fn(k % ncopies)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / calls


def measure_interleaved(fns, reps, ncopies, passes):
    """Best-of-`passes` measure() for each fn, the passes interleaved across
    the fns so clock or thermal drift does not favour the one timed first."""
    best = [float("inf")] * len(fns)
    for _ in range(passes):
        for i, fn in enumerate(fns):
            best[i] = min(best[i], measure(fn, reps, ncopies))
    return best


def measure_single(fn, reps, flush):
    """One call at a time after a 512 MB L2 flush (single-call latency)."""
    times = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(min(reps, 10)):
        flush.zero_()
        e0.record()
        fn(0)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    return statistics.median(times)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", default="dgemv,dgemv_t,zgemv,zgemv_c,sgemv,sgemv_t,cgemv,cgemv_c,"
                                     "cgemv_t,zgemv_t,dsymv,dsymv_u,zhemv,zhemv_u,ssymv,ssymv_u,chemv,chemv_u")
    ap.add_argument("--sizes", default="1024,2048,4096,8192,12288,16383,16384,20480,24576,32768,40960,49152,60000")
    ap.add_argument("--max-gb", type=float, default=60.0)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("--passes", type=int, default=3, help="interleaved timing passes (best kept)")
    ap.add_argument("--ld-pad", type=int, default=0, help="leading dimension = round_up(m, 32) + this")
    ap.add_argument("--ab-table", action="store_true",
                    help="also time each point with the tuning table cleared (built-in rules only)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    lib = _lib.load()
    cub = None if args.no_cublas else Cublas()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    rows = []
    out = open(args.out, "w") if args.out else None
    for opname in args.ops.split(","):
        tag, family, op, herm = OPS[opname]
        p = precision(tag)
        for n in [int(s) for s in args.sizes.split(",")]:
            m = n
            ld = -(-m // 32) * 32 + args.ld_pad
            if n * ld * p.element_bytes > args.max_gb * 1e9:
                continue
            mat_alloc = n * ld * p.element_bytes
            ncop = max(1, min(64, -(-(1 << 30) // mat_alloc)))
            As = []
            for _ in range(ncop):
                A = torch.empty(n, ld, dtype=p.torch_dtype, device=dev)
                (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1)
                As.append(A)
            x = torch.empty(n, dtype=p.torch_dtype, device=dev)
            y = torch.empty(n, dtype=p.torch_dtype, device=dev)
            (torch.view_as_real(x) if p.is_complex else x).uniform_(-1, 1)
            sh = torch.cuda.current_stream().cuda_stream
            one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)
            if family == "symv":
                name = {("s", False): "ssymv", ("d", False): "dsymv", ("c", True): "chemv", ("z", True): "zhemv"}[(tag, herm)]
                f = getattr(lib, f"kblas_{name}_async")

                def ours(k):
                    assert f(op.encode(), n, one, As[k].data_ptr(), ld, x.data_ptr(), 1, zero, y.data_ptr(), 1, sh) == 0
            else:
                f = getattr(lib, f"kblas_{tag}gemv_async")

                def ours(k):
                    assert f(op.encode(), m, n, one, As[k].data_ptr(), ld, x.data_ptr(), 1, zero, y.data_ptr(), 1, sh) == 0

            nbytes = alg_bytes(tag, family, m, n, op)
            fns = [ours]
            saved_table = None
            if args.ab_table:
                from paper_1410_1726_b200 import tuner

                saved_table = tuner.table()
                # the rules-only arm is the same call timed with the table
                # cleared for its whole window (below)
                fns.append(ours)
            y2 = None
            have_cublas = cub is not None and cub.lib is not None
            if have_cublas:
                y2 = torch.empty_like(y)

                def theirs(k):
                    cub.call(tag, family, op, herm, m, n, As[k].data_ptr(), ld, x.data_ptr(), y2.data_ptr(), sh)

                have_cublas = cub.call(tag, family, op, herm, m, n, As[0].data_ptr(), ld, x.data_ptr(), y2.data_ptr(),
                                       sh)
                if have_cublas:
                    fns.append(theirs)
            best = [float("inf")] * len(fns)
            for _ in range(args.passes):
                for i, fn in enumerate(fns):
                    rules_arm = saved_table is not None and i == 1
                    if rules_arm:
                        lib.kblas_tune_clear()
                    try:
                        best[i] = min(best[i], measure(fn, args.reps, ncop))
                    finally:
                        if rules_arm:
                            tuner.restore(saved_table)
            ms = best[0]
            sms = measure_single(ours, args.reps, flush)
            plan = _lib.last_plan()
            row = {"op": opname, "n": n, "ld": ld, "ms": round(ms, 5), "gbs": round(nbytes / ms / 1e6, 1),
                   "pct_peak": round(100 * nbytes / ms / 1e6 / PEAK, 1), "single_ms": round(sms, 5),
                   "single_gbs": round(nbytes / sms / 1e6, 1), "copies": ncop, "plan": plan}
            if saved_table is not None:
                lib.kblas_tune_clear()
                ours(0)
                row["rules_plan"] = _lib.last_plan()
                tuner.restore(saved_table)
                row["rules_gbs"] = round(nbytes / best[1] / 1e6, 1)
                row["table_gain"] = round(best[1] / ms, 3)
            if have_cublas:
                cms = best[-1]
                row["cublas_gbs"] = round(nbytes / cms / 1e6, 1)
                row["speedup_vs_cublas"] = round(cms / ms, 3)
                ours(0)
                theirs(0)  # same operand copy on both sides
                scale = float((y2.abs().max()).item()) or 1.0
                row["rel_diff_vs_cublas"] = float(((y - y2).abs().max() / scale).item())
            rows.append(row)
            line = json.dumps(row)
            print(line, flush=True)
            if out:
                out.write(line + "\n")
                out.flush()
            del As, x, y
            torch.cuda.empty_cache()
    if out:
        out.close()


if __name__ == "__main__":
    main()
