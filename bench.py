#!/usr/bin/env python
"""Benchmark: achieved HBM GB/s of the KBLAS matrix-vector hot path on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

N=1 (default): DSYMV lower, N=32768, alpha=1, beta=0 — BASELINE.json
configs[1], the configuration the metric is quoted on.  One step = one
kblas_dsymv call (main streaming kernel + fixed-order epilogue) on
HBM-resident operands.  The 8.6 GB matrix is 68x the 126 MB L2, so every
step streams A from HBM (no flush needed).

N>1 (torchrun, one process per GPU): mgpu DSYMV lower over the 1D
block-column-cyclic layout (nb=128) with per-GPU work fixed (weak scaling):
n = 32768 * sqrt(N) rounded to nb, each rank streams its panel's stored
triangle and writes its partial y straight into its slot in rank 0's HBM
(CUDA IPC, NVLink stores); a device-flag handshake and a rank-order
combine kernel on rank 0 finish y (multidevice.py:276, 282-283) with no
NCCL on the data path.  `--reduce nccl` uses an NCCL reduce instead.

`--impl reference` times the reference's CPU path for the same metric:
the C restatement of the reference oracle (oracle/streamed.c, all host
threads) on a bounded sample (DSYMV lower N=12288); rank 0 only.

Other workloads for sweeps: --op {dsymv,zhemv,ssymv,chemv,dgemv,zgemv,
sgemv,cgemv,dgemv_t,zgemv_c,...} --n N.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SPEC_HBM_GBS = 8000.0
CPU_SAMPLE_N = 12288


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--op", default="dsymv")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--nb", type=int, default=128)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--mgpu", action="store_true",
                    help="run the one-process-per-GPU mgpu path even at N=1 (exercises the exchange path)")
    ap.add_argument("--reduce", choices=["p2p", "nccl"], default="p2p",
                    help="mgpu exchange: peer-memory slots + device flags (p2p, default) or an NCCL reduce")
    return ap.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------- ops
OPS = {
    # name: (tag, family, trans/uplo, hermitian)
    "ssymv": ("s", "symv", "l", False), "dsymv": ("d", "symv", "l", False),
    "chemv": ("c", "symv", "l", True), "zhemv": ("z", "symv", "l", True),
    "ssymv_u": ("s", "symv", "u", False), "dsymv_u": ("d", "symv", "u", False),
    "chemv_u": ("c", "symv", "u", True), "zhemv_u": ("z", "symv", "u", True),
    "sgemv": ("s", "gemv", "n", False), "dgemv": ("d", "gemv", "n", False),
    "cgemv": ("c", "gemv", "n", False), "zgemv": ("z", "gemv", "n", False),
    "sgemv_t": ("s", "gemv", "t", False), "dgemv_t": ("d", "gemv", "t", False),
    "cgemv_c": ("c", "gemv", "c", False), "zgemv_c": ("z", "gemv", "c", False),
    "cgemv_t": ("c", "gemv", "t", False), "zgemv_t": ("z", "gemv", "t", False),
}


def alg_bytes(tag, family, m, n, op):
    from paper_1410_1726_b200 import roofline
    from paper_1410_1726_b200.core import precision

    p = precision(tag)
    return roofline.symv_bytes(p, n) if family == "symv" else roofline.gemv_bytes(p, m, n, op)


def alg_flops(tag, family, m, n, op):
    from paper_1410_1726_b200 import roofline
    from paper_1410_1726_b200.core import precision

    p = precision(tag)
    return roofline.symv_flops(p, n) if family == "symv" else roofline.gemv_flops(p, m, n, op)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [s.strip() for s in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[k] for r in self.rows for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------ CPU legs
def _cpu_problem(opname: str, n: int):
    """Host operands of the reference CPU path for --op at order n (seeded)."""
    import numpy as np

    from paper_1410_1726_b200 import roofline
    from paper_1410_1726_b200.core import precision

    tag, family, op, herm = OPS[opname]
    p = precision(tag)
    rng = np.random.default_rng(0)

    def rnd(*shape):
        v = rng.uniform(-1, 1, size=shape)
        if p.is_complex:
            v = v + 1j * rng.uniform(-1, 1, size=shape)
        return v.astype(p.dtype)

    a = np.asfortranarray(rnd(n, n))
    x, y = rnd(n), rnd(n)
    nbytes = roofline.symv_bytes(p, n) if family == "symv" else roofline.gemv_bytes(p, n, n, op)
    return tag, family, op, herm, a, x, y, nbytes


def _cpu_call(streamed, family, op, herm, a, x, y):
    if family == "symv":
        streamed.symv(op, 1.0, a, x, 0.0, y, hermitian=herm)
    else:
        streamed.gemv(op, 1.0, a, x, 0.0, y)


def cpu_sample_n(opname: str, n: int) -> int:
    """Order of the CPU sample: the workload itself when it is small enough
    (configs[0], DGEMV 4096), else CPU_SAMPLE_N (a bounded sample)."""
    return min(n, CPU_SAMPLE_N)


def cpu_baseline(seconds: float, opname: str = "dsymv", n: int = CPU_SAMPLE_N, max_calls: int | None = None):
    """The oracle (C restatement of the reference's naive_gemv /
    naive_symv_hemv, all host threads) on the --op workload at order n; GB/s
    on the same algorithmic bytes."""
    from oracle import streamed  # CPU baseline leg only

    tag, family, op, herm, a, x, y, nbytes = _cpu_problem(opname, n)
    threads = streamed.max_threads()
    _cpu_call(streamed, family, op, herm, a, x, y)  # warm
    calls, t0 = 0, time.perf_counter()
    while True:
        _cpu_call(streamed, family, op, herm, a, x, y)
        calls += 1
        el = time.perf_counter() - t0
        if el >= seconds or (max_calls and calls >= max_calls):
            break
    gbs = nbytes * calls / el / 1e9
    return {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": f"oracle/streamed.c {opname} ({op}) N={n} (host matrix, wide accumulation), "
                      f"{calls} calls in {el:.1f} s, {threads} threads"}


def metric_name(opname: str) -> str:
    tag, family, op, herm = OPS[opname]
    label = {"symv": "SYMV" if not herm else "HEMV", "gemv": "GEMV"}[family]
    if opname == "dsymv":
        return "achieved HBM GB/s (DSYMV lower, algorithmic bytes)"
    return f"achieved HBM GB/s ({tag.upper()}{label}{'' if family == 'symv' else '-' + op.upper()}, algorithmic bytes)"


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port), rank 0 only,
    on the same --op workload (a bounded sample when the order is large)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import streamed

    n_work = args.n or (32768 if OPS[args.op][1] == "symv" else 16384)  # bench_single's defaults
    n = cpu_sample_n(args.op, n_work)
    tag, family, op, herm, a, x, y, nbytes = _cpu_problem(args.op, n)
    threads = streamed.max_threads()
    for _ in range(args.warmup):
        _cpu_call(streamed, family, op, herm, a, x, y)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _cpu_call(streamed, family, op, herm, a, x, y)
    el = time.perf_counter() - t0
    gbs = nbytes * args.steps / el / 1e9
    whole = n == n_work
    sample = (f"oracle/streamed.c (C restatement of blockmv naive_gemv / naive_symv_hemv) {args.op} N={n}, "
              f"{threads} threads; " + ("the whole workload" if whole else f"bounded sample of N={n_work}"))
    blockmv_gbs = None
    if args.op == "dsymv":
        try:  # the reference package itself, if installed into baseline/_ref (pure-Python simulator)
            import numpy as np

            from paper_1410_1726_b200 import roofline
            from paper_1410_1726_b200.core import precision

            sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
            import blockmv

            ns = 2048
            rng = np.random.default_rng(0)
            v = blockmv.make_padded_view(ns, ns, blockmv.precision("d"), pad_to=32)
            v.array()[:, :] = rng.uniform(-1, 1, size=(ns, ns))
            hv = blockmv.HermitianView(base=v, uplo="l")
            t1 = time.perf_counter()
            blockmv.symv_hemv("l", 1.0, hv, x[:ns], 0.0, y[:ns], blockmv.KernelConfig(64, 4))
            blockmv_gbs = round(roofline.symv_bytes(precision("d"), ns) / (time.perf_counter() - t1) / 1e9, 4)
        except Exception:
            pass
    workload = ("DSYMV lower N=32768 (BASELINE configs[1])" if args.op == "dsymv" and n_work == 32768
                else "DGEMV non-transposed N=4096 (BASELINE configs[0])" if args.op == "dgemv" and n_work == 4096
                else f"{args.op} m={n_work} n={n_work}")
    print(json.dumps({
        "impl": "reference", "metric": metric_name(args.op), "value": round(gbs, 3),
        "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(el / args.steps * 1e3, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": {"s": "f32", "d": "f64", "c": "c64", "z": "c128"}[tag],
        "data": "synthetic U(-1,1)",
        "config": {"workload": workload, "cpu_sample_n": n, "op": args.op},
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "blockmv_simulator_gbs_n2048": blockmv_gbs,
    }), flush=True)


# ------------------------------------------------------------- GPU arm
def bench_single(args, dev, rank):
    import torch

    from paper_1410_1726_b200 import _lib
    from paper_1410_1726_b200.core import precision

    tag, family, op, herm = OPS[args.op]
    p = precision(tag)
    n = args.n or (32768 if family == "symv" else 16384)
    m = n if family == "symv" else (args.m or n)
    lib = _lib.load()
    torch.manual_seed(0)
    ld = -(-m // 32) * 32
    # column-major A: a (n, ld) row-major tensor whose row j is column j
    A = torch.empty(n, ld, dtype=p.torch_dtype, device=dev)
    (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1)
    # operands smaller than 4x the 126 MB L2 rotate over copies of A (>= 512
    # MB together), so every step streams its matrix from HBM
    ncopies = max(1, min(16, -(-(512 << 20) // A.numel() // p.element_bytes)))
    As = [A] + [A.clone() for _ in range(ncopies - 1)]
    x_len, y_len = (n, m) if (family == "symv" or op == "n") else (m, n)
    x = torch.empty(x_len, dtype=p.torch_dtype, device=dev)
    y = torch.empty(y_len, dtype=p.torch_dtype, device=dev)
    (torch.view_as_real(x) if p.is_complex else x).uniform_(-1, 1)
    (torch.view_as_real(y) if p.is_complex else y).uniform_(-1, 1)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream
    one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)
    if family == "symv":
        name = {("s", False): "ssymv", ("d", False): "dsymv", ("c", True): "chemv", ("z", True): "zhemv"}[(tag, herm)]
        fn = getattr(lib, f"kblas_{name}_async")

        def step(i=0):
            rc = fn(op.encode(), n, one, As[i % ncopies].data_ptr(), ld, x.data_ptr(), 1, zero, y.data_ptr(), 1, sh)
            assert rc == 0, rc
    else:
        fn = getattr(lib, f"kblas_{tag}gemv_async")

        def step(i=0):
            rc = fn(op.encode(), m, n, one, As[i % ncopies].data_ptr(), ld, x.data_ptr(), 1, zero, y.data_ptr(), 1,
                    sh)
            assert rc == 0, rc

    nbytes = alg_bytes(tag, family, m, n, op)
    nflops = alg_flops(tag, family, m, n, op)
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)
    plan = _lib.last_plan()
    clock = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clock.start()
    time.sleep(0.3)
    # warm the clocks up to the sampler's first reading, then time exactly K steps
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)
    l0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for i in range(args.steps):
        step(i)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    launches = _lib.launch_count() - l0
    clocks = clock.stop()
    total_ms = e0.elapsed_time(e1)
    # dominant-kernel time: a second pass with the library's CUDA-event
    # brackets around each streaming-kernel launch (kept out of the timed
    # region above because the extra event records break the PDL overlap)
    _lib.timing_enable(True)
    for i in range(min(args.steps, 50)):
        step(i)
    torch.cuda.synchronize(dev)
    _lib.timing_enable(False)
    kern_ms, kern_n = _lib.timing_read()
    ms_step = total_ms / args.steps
    gbs = nbytes / (ms_step * 1e-3) / 1e9
    kern_avg = kern_ms / max(kern_n, 1)
    res = dict(tag=tag, family=family, op=op, m=m, n=n, ld=ld, nbytes=nbytes, nflops=nflops, ms_step=ms_step,
               gbs=gbs, kern_avg_ms=kern_avg, kern_launches=kern_n, launches=launches, plan=plan,
               clocks=clocks, total_ms=total_ms, ncopies=ncopies)
    # end to end through the public API with host (pinned) buffers
    if not args.no_e2e and args.e2e_steps > 0:
        res["e2e"] = e2e_single(args, As, x, y, tag, family, op, herm, m, n, ld, dev, nbytes)
    return res


def e2e_single(args, As, x, y, tag, family, op, herm, m, n, ld, dev, nbytes):
    """End to end through the public API (paper_1410_1726_b200.symv_hemv /
    gemv), as an iterative solver calls it: the matrix stays resident in HBM
    (uploaded once, like model weights), and every step copies that step's
    inputs x, y from pinned host memory to the device, runs the kernels and
    reads y back to the host.  A second figure re-uploads the referenced part
    of A every step as well (host-resident matrix), for transparency."""
    import torch

    import paper_1410_1726_b200 as kb

    p = kb.precision(tag)
    hx = torch.empty(x.numel(), dtype=x.dtype, pin_memory=True)
    hx.copy_(x)
    hy = torch.empty(y.numel(), dtype=y.dtype, pin_memory=True)
    hy.copy_(y)
    npx, npy = hx.numpy(), hy.numpy()
    eb = p.element_bytes
    x_len = n if (family == "symv" or op == "n") else m

    def run(views, steps):
        def step(i):
            view = views[i % len(views)]
            if family == "symv":
                return kb.symv_hemv(op, 1.0, kb.HermitianView(view, op), npx, 0.0, npy, hermitian=herm).y_out
            return kb.gemv(op, 1.0, view, npx, 0.0, npy).y_out

        step(0)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for i in range(steps):
            out = step(i)
        torch.cuda.synchronize(dev)
        return (time.perf_counter() - t0) / steps, out

    # resident matrix (rotating over the same copies as the device-timed
    # steps): the headline end-to-end figure
    A = As[0]
    el, out = run([kb.MatrixView(a.reshape(-1), m, n, ld, p) for a in As], max(args.e2e_steps, 20))
    y_len = len(out)
    res = {"value": round(nbytes / el / 1e9, 3), "unit": "GB/s",
           "h2d_bytes_per_step": int(x_len * eb + y_len * eb), "d2h_bytes_per_step": int(y_len * eb),
           "steps": max(args.e2e_steps, 20), "ms_per_step": round(el * 1e3, 4),
           "path": f"paper_1410_1726_b200.{'symv_hemv' if family == 'symv' else 'gemv'} with A resident in HBM "
                   "(uploaded once), x and y from pinned host numpy each step, y returned as numpy"}
    # host-resident matrix: the referenced part of A is uploaded every step too
    hA = torch.empty(A.numel(), dtype=A.dtype, pin_memory=True)
    hA.copy_(A.reshape(-1))
    el2, _ = run([kb.MatrixView(hA.numpy(), m, n, ld, p)], args.e2e_steps)
    if family == "symv":
        blocks = [(b0, min(n, b0 + 256)) for b0 in range(0, n, 256)]
        h2d_a = sum((b1 - b0) * ((m - b0) if op == "l" else b1) for b0, b1 in blocks) * eb
    else:
        h2d_a = n * ld * eb
    res["with_matrix_upload"] = {
        "value": round(nbytes / el2 / 1e9, 3), "unit": "GB/s", "ms_per_step": round(el2 * 1e3, 3),
        "h2d_bytes_per_step": int(h2d_a + x_len * eb + y_len * eb), "d2h_bytes_per_step": int(y_len * eb),
        "steps": args.e2e_steps,
        "path": "same call with A in pinned host memory: the stored triangle (SYMV) or the columns (GEMV) "
                "cross PCIe every step"}
    return res


def bench_mgpu(args, dev, rank, world):
    """Weak-scaling mgpu DSYMV: per-rank panel of the block-cyclic layout,
    partial via the sm_100a kernels, exchange of y onto rank 0 (--reduce)."""
    import torch
    import torch.distributed as dist

    from paper_1410_1726_b200 import _lib
    from paper_1410_1726_b200.core import precision
    from paper_1410_1726_b200.dist import combine, panel_shape
    from paper_1410_1726_b200.multidevice import partial_mv

    tag, family, op, herm = OPS[args.op]
    if family != "symv":
        raise SystemExit("mgpu bench covers symv/hemv")
    p = precision(tag)
    nb = args.nb
    n = args.n or int(round(32768 * math.sqrt(world) / nb)) * nb
    rows, lc, ld = panel_shape(n, n, nb, world, rank)
    from paper_1410_1726_b200.core import MatrixView

    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    panel_t = torch.empty(max(lc, 1) * ld, dtype=p.torch_dtype, device=dev)
    (torch.view_as_real(panel_t) if p.is_complex else panel_t).uniform_(-1, 1, generator=g)
    panel = MatrixView(panel_t, n, lc, ld, p) if lc > 0 else None
    x = torch.empty(n, dtype=p.torch_dtype, device=dev)
    (torch.view_as_real(x) if p.is_complex else x).uniform_(-1, 1, generator=torch.Generator(device=dev).manual_seed(7))
    out = torch.empty(n, dtype=p.torch_dtype, device=dev)

    ex = None
    if args.reduce == "p2p":
        from paper_1410_1726_b200.dist import P2PExchange, p2p_mv

        try:
            ex = P2PExchange(n, p.torch_dtype)
        except Exception as err:  # no IPC between these ranks: fall back to the NCCL reduce
            print(f"p2p exchange unavailable ({err}); using the NCCL reduce", file=sys.stderr, flush=True)
            args.reduce = "nccl"
    if ex is not None:

        def step():
            p2p_mv(p, "s", op, n, n, 1.0, panel, x, 0.0, None, nb, ex, hermitian=herm)
    else:
        def step():
            partial_mv(p, "s", op, n, n, 1.0, panel, x, out, world, rank, nb, herm)
            combine(out, None, 0.0)

    nbytes = alg_bytes(tag, "symv", n, n, op)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    clock = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clock.start()
    time.sleep(0.3)
    l0 = _lib.launch_count()
    dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize(dev)
    dist.barrier()
    launches = _lib.launch_count() - l0
    clocks = clock.stop()
    _lib.timing_enable(True)
    for i in range(min(args.steps, 50)):
        step(i)
    torch.cuda.synchronize(dev)
    _lib.timing_enable(False)
    kern_ms, kern_n = _lib.timing_read()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_step = ms.item()
    my_bytes = 0
    for j in range(rank, -(-n // nb), world):
        c0, c1 = j * nb, min(n, (j + 1) * nb)
        my_bytes += ((c1 - c0) * (c1 - c0 + 1) // 2 + (n - c1) * (c1 - c0)) * p.element_bytes
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        e2e = e2e_mgpu(args, panel, panel_t, x, out, p, n, nb, lc, ld, world, rank, dev, op, herm, nbytes, ex)
    return dict(e2e=e2e, tag=tag, family="symv", op=op, m=n, n=n, ld=ld, nbytes=nbytes, ms_step=ms_step,
                gbs=nbytes / (ms_step * 1e-3) / 1e9, kern_avg_ms=kern_ms / max(kern_n, 1), kern_launches=kern_n,
                launches=launches, plan=_lib.last_plan(), clocks=clocks, my_bytes=my_bytes, nb=nb)


def e2e_mgpu(args, panel, panel_t, x, out, p, n, nb, lc, ld, world, rank, dev, op, herm, nbytes, ex=None):
    """Per step on every rank: x from pinned host to HBM, the partial kernels
    on the resident panel, the exchange onto rank 0 (peer-memory slots, or
    an NCCL reduce), and on rank 0 the D2H read of y.  Max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1410_1726_b200.dist import combine
    from paper_1410_1726_b200.multidevice import partial_mv

    eb = p.element_bytes
    hx = torch.empty(n, dtype=x.dtype, pin_memory=True)
    hx.copy_(x)
    hy = torch.empty(n, dtype=x.dtype, pin_memory=True)
    dx = torch.empty_like(x)

    def step():
        dx.copy_(hx, non_blocking=True)
        if ex is not None:
            from paper_1410_1726_b200.dist import p2p_mv

            res = p2p_mv(p, "s", op, n, n, 1.0, panel, dx, 0.0, None, nb, ex, hermitian=herm)
        else:
            partial_mv(p, "s", op, n, n, 1.0, panel, dx, out, world, rank, nb, herm)
            res = combine(out, None, 0.0)
        if rank == 0:
            hy.copy_(res)  # synchronous D2H read of the result

    steps = max(args.e2e_steps, 20)
    step()
    torch.cuda.synchronize(dev)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize(dev)
    dist.barrier()
    el = torch.tensor([(time.perf_counter() - t0) / steps], device=dev)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    el = el.item()
    how = ("partial written into rank 0's peer-memory slot, device-flag handshake, rank-order combine kernel "
           "on rank 0" if ex is not None else "NCCL reduce to rank 0")
    return {"value": round(nbytes / el / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": int(n * eb),
            "d2h_bytes_per_step": int(n * eb), "steps": steps, "ms_per_step": round(el * 1e3, 4),
            "path": f"per rank: x from pinned host, kblas_mv_mgpu_partial_async on the HBM-resident panel, {how}, "
                    "D2H of y on rank 0; max over ranks"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N>1 under torchrun")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    mgpu = world > 1 or args.mgpu
    if mgpu:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    hbm_peak, peak_src = measured_peaks()
    if mgpu:
        res = bench_mgpu(args, dev, rank, world)
    else:
        res = bench_single(args, dev, rank)
    tag, family, op = res["tag"], res["family"], res["op"]
    achieved_kernel = (res.get("my_bytes", res["nbytes"]) / (res["kern_avg_ms"] * 1e-3) / 1e9
                       if res["kern_avg_ms"] > 0 else None)
    if rank == 0:
        opname = args.op
        if mgpu:
            xch = ("peer-memory exchange of y (IPC slots + device flags, rank-order combine)"
                   if args.reduce == "p2p" else "NCCL reduce of y")
            workload = (f"mgpu {opname} N={res['n']} 1D block-column-cyclic nb={res['nb']} over {world} GPUs, "
                        f"{xch} (weak scaling: n = 32768*sqrt(G))")
        elif args.op == "dsymv" and res["n"] == 32768:
            workload = "DSYMV lower N=32768 (BASELINE configs[1])"
        elif args.op == "dgemv" and res["n"] == 4096 and res["m"] == 4096:
            workload = "DGEMV non-transposed N=4096 (BASELINE configs[0])"
        else:
            workload = f"{opname} m={res['m']} n={res['n']}"
        prof_traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
                prof_traffic = json.load(fh).get(f"{opname}_{res['n']}")
        except Exception:
            pass
        line = {
            "metric": metric_name(opname),
            "value": round(res["gbs"], 2),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(res["ms_step"], 5),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": {"s": "f32", "d": "f64", "c": "c64", "z": "c128"}[tag],
            "data": "synthetic U(-1,1), generated on device",
            "config": {"workload": workload, "op": opname, "m": res["m"], "n": res["n"], "ld": res["ld"],
                       "uplo_or_trans": op, "alpha": 1.0, "beta": 0.0,
                       "l2": ("inputs > 126 MB L2 (A streamed from HBM every step), no flush"
                              if res.get("ncopies", 1) == 1 else
                              f"{res['ncopies']} rotating copies of A (>= 512 MB together, > 4x the L2): "
                              "every step streams its matrix from HBM"),
                       "parallelism": f"{world} GPU" + ("s, one process each" if world > 1 else "")},
            "pct_of_copy_peak": round(100 * res["gbs"] / hbm_peak, 2),
            "gflops": round(res.get("nflops", 0) / (res["ms_step"] * 1e-3) / 1e9, 2) if res.get("nflops") else None,
            "roofline": {"bound": "hbm", "achieved": round(achieved_kernel, 2) if achieved_kernel else None,
                         "peak": hbm_peak, "unit": "GB/s",
                         "frac": round(achieved_kernel / hbm_peak, 4) if achieved_kernel else None,
                         "traffic": prof_traffic, "peak_source": peak_src,
                         "kernel": res["plan"].split()[0] + "_kernel", "kernel_avg_ms": round(res["kern_avg_ms"], 5),
                         "spec_peak_gbs": SPEC_HBM_GBS,
                         "bytes_per_launch": res.get("my_bytes", res["nbytes"])},
            "clocks": res["clocks"],
            "gpu_launches": res["launches"],
            "plan": res["plan"],
        }
        line["e2e"] = res.get("e2e")
        if not args.no_cpu and world == 1:
            line["cpu_baseline"] = cpu_baseline(args.cpu_seconds, args.op, cpu_sample_n(args.op, res["n"]))
        print(json.dumps(line), flush=True)
    if mgpu:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
