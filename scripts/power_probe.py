#!/usr/bin/env python
"""Sustained-load probe: back-to-back SYMV/HEMV calls on one operand for a
few seconds, per-call device time (CUDA events) next to nvidia-smi samples
of SM clock, board power and throttle reasons (every 100 ms).  Shows
whether a kernel slows down as the board reaches its power cap.

    python scripts/power_probe.py --ops dsymv,zhemv --n 100000 --seconds 4
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import OPS, alg_bytes  # noqa: E402
from paper_1410_1726_b200 import _lib  # noqa: E402
from paper_1410_1726_b200.core import precision  # noqa: E402

FIELDS = "timestamp,clocks.sm,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown"


def sampler(rows, stop):
    p = subprocess.Popen(["nvidia-smi", f"--query-gpu={FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                          "-i", "0"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    for line in p.stdout:
        rows.append((time.perf_counter(), [s.strip() for s in line.split(",")]))
        if stop.is_set():
            break
    p.terminate()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", default="dsymv,zhemv")
    ap.add_argument("--n", type=int, default=100000)
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--idle", type=float, default=3.0, help="idle seconds before each op")
    args = ap.parse_args()
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream().cuda_stream
    for opname in args.ops.split(","):
        tag, family, op, herm = OPS[opname]
        p = precision(tag)
        name = {("s", False): "ssymv", ("d", False): "dsymv", ("c", True): "chemv", ("z", True): "zhemv"}[(tag, herm)]
        fn = getattr(lib, f"kblas_{name}_async")
        n = args.n
        A = torch.empty(n, n, dtype=p.torch_dtype, device=dev)
        (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1)
        x = torch.ones(n, dtype=p.torch_dtype, device=dev)
        y = torch.empty(n, dtype=p.torch_dtype, device=dev)
        one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)
        call = lambda: fn(op.encode(), n, one, A.data_ptr(), n, x.data_ptr(), 1, zero, y.data_ptr(), 1, st)
        call()
        torch.cuda.synchronize()
        time.sleep(args.idle)
        rows, stop = [], threading.Event()
        th = threading.Thread(target=sampler, args=(rows, stop), daemon=True)
        th.start()
        time.sleep(0.3)
        evs = []
        t0 = time.perf_counter()
        t_host = []
        while time.perf_counter() - t0 < args.seconds:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            call()
            e1.record()
            evs.append((e0, e1))
            t_host.append(time.perf_counter() - t0)
            if len(evs) % 8 == 0:
                e1.synchronize()
        torch.cuda.synchronize()
        stop.set()
        th.join(timeout=3)
        ms = [a.elapsed_time(b) for a, b in evs]
        nbytes = alg_bytes(tag, "symv", n, n, op)
        k = max(1, len(ms) // 8)
        first, last = ms[:k], ms[-k:]
        sm = [float(r[1]) for _, r in rows if r[1].replace(".", "").isdigit()]
        pw = [float(r[2]) for _, r in rows if r[2].replace(".", "").isdigit()]
        cap = sum(1 for _, r in rows if r[3] == "Active")
        print(json.dumps({
            "op": opname, "n": n, "calls": len(ms),
            "gbs_first_eighth": round(nbytes / (statistics.median(first) * 1e-3) / 1e9, 1),
            "gbs_last_eighth": round(nbytes / (statistics.median(last) * 1e-3) / 1e9, 1),
            "gbs_median": round(nbytes / (statistics.median(ms) * 1e-3) / 1e9, 1),
            "sm_mhz_min_median_max": [min(sm), statistics.median(sm), max(sm)] if sm else None,
            "power_w_median_max": [statistics.median(pw), max(pw)] if pw else None,
            "sw_power_cap_samples": f"{cap}/{len(rows)}",
            "per_call_ms_series": [round(v, 3) for v in ms[:: max(1, len(ms) // 40)]],
            "sm_mhz_series": sm[:: max(1, len(sm) // 40)]}), flush=True)
        del A
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
