#!/usr/bin/env python
"""Benchmark: achieved HBM GB/s of the KBLAS matrix-vector hot path on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
    (N > 1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N)

Default workload at EVERY N (the north_star's scaling claim, BASELINE.json
configs[4]): mgpu DSYMV lower, N = 100000, nb = 128, 1D block-column-cyclic
over the N GPUs, one process per GPU, STRONG scaling (the same 40 GB
triangle at every N, so the driver's per-N values give T(1) / (N T(N))
directly).  One step = one distributed y = A x: every rank streams its
panel's stored triangle through the sm_100a SYMV kernel and the partial y
vectors are summed onto rank 0 (multidevice.py:183-284).  Two exchanges
are timed in the same run:

  p2p   (headline) each rank's SYMV epilogue stores its partial straight
        into its slot in rank 0's HBM (CUDA IPC, NVLink stores) and rank 0's
        epilogue adds the slots in rank order (dist.P2PExchange);
  nccl  the partial kernels, then an NCCL reduce(sum) onto rank 0
        (dist.combine) -- the north_star's "NCCL reduce over NVLink".

`value` is 40.0 GB of algorithmic bytes (b (n(n+1)/2 + 3n))
divided by the step time, timed with CUDA events between barriers and
taken as the MAX over ranks.  Per rank the line also reports the streaming
kernel's time, the partial-only step time (no exchange) and hence the
exchange cost.  A ZHEMV N=100000 block follows (same layout; 160 GB, so at
N=1 it needs the whole HBM), and at N=1 two single-GPU blocks keep the
other BASELINE configs driver-measured: configs[1] DSYMV L N=32768 (with
cuBLAS dsymv on the same buffers) and configs[0] DGEMV N=4096.

`--impl reference` times the reference's CPU path for the same workload:
the C restatement of the reference oracle (oracle/streamed.c, naive_symv_hemv
from the stored triangle, all host threads) on a host copy of an N=100000
operand; rank 0 only, the other ranks exit 0.

Legacy single-op mode for sweeps: --op {dsymv,zhemv,ssymv,chemv,dgemv,zgemv,
sgemv,cgemv,dgemv_t,zgemv_c,...} [--n N] (single GPU unless --mgpu / N>1).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SPEC_HBM_GBS = 8000.0
CPU_SAMPLE_N = 12288
NS_N, NS_NB = 100000, 128  # BASELINE configs[4]
NS_METRIC = "mgpu DSYMV lower N=100000 achieved HBM GB/s (algorithmic bytes, strong scaling over G GPUs)"
NS_WORKLOAD = ("mgpu DSYMV lower N=100000, nb=128, 1D block-column-cyclic over G GPUs, one process per GPU "
               "(BASELINE configs[4])")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--op", default=None, help="legacy single-op mode (sweeps); default: the configs[4] workload")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--nb", type=int, default=NS_NB)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="north-star mode: skip the ZHEMV / configs[1] / configs[0] blocks")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--mgpu", action="store_true",
                    help="legacy mode: run the one-process-per-GPU mgpu path even at N=1")
    ap.add_argument("--reduce", choices=["p2p", "nccl"], default="p2p",
                    help="legacy mgpu mode: the exchange (north-star mode times both)")
    return ap.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


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
DTYPE_NAME = {"s": "f32", "d": "f64", "c": "c64", "z": "c128"}


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


def traffic_of(key: str):
    """ncu dram bytes per launch of the dominant kernel for this workload
    (profiles/traffic.json, from `ncu --set full` captures)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh).get(key)
    except Exception:
        return None


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
def _rnd(rng, p, *shape):
    v = rng.uniform(-1, 1, size=shape)
    if p.is_complex:
        v = v + 1j * rng.uniform(-1, 1, size=shape)
    return v.astype(p.dtype)


def host_symv_operand(tag: str, n: int):
    """Host operand of the reference CPU path: an n x n column-major buffer
    whose stored (lower) triangle is filled (OpenMP, counter-based
    generator); the other triangle is never touched, so only ~half the
    pages are ever backed."""
    import numpy as np

    from oracle import streamed

    dt = streamed.DTYPES[tag]
    buf = np.empty(n * n, dtype=dt)
    rc = streamed.load().oracle_gen_fill_tri(tag.encode(), b"l", n, 5, n, buf.ctypes.data, n, host_threads())
    assert rc == 0
    return buf.reshape(n, n).T  # column-major view


def cpu_symv_n(n_work: int, tag: str = "d") -> int:
    """Largest order <= n_work whose host operand fits in ~45 % of RAM."""
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except Exception:
        avail = 64 << 30
    eb = {"s": 4, "d": 8, "c": 8, "z": 16}[tag]
    n = n_work
    while n > 4096 and n * n * eb / 2 > 0.45 * avail:
        n = int(n * 0.9) // 128 * 128
    return n


def _cpu_problem(opname: str, n: int):
    """Host operands of the reference CPU path for --op at order n (seeded)."""
    import numpy as np

    from paper_1410_1726_b200 import roofline
    from paper_1410_1726_b200.core import precision

    tag, family, op, herm = OPS[opname]
    p = precision(tag)
    rng = np.random.default_rng(0)
    if family == "symv" and op == "l" and n > 16384:
        a = host_symv_operand(tag, n)
    else:
        a = np.asfortranarray(_rnd(rng, p, n, n))
    x, y = _rnd(rng, p, n), _rnd(rng, p, n)
    nbytes = roofline.symv_bytes(p, n) if family == "symv" else roofline.gemv_bytes(p, n, n, op)
    return tag, family, op, herm, a, x, y, nbytes


def host_threads() -> int:
    """Every host core this process may run on.  Passed explicitly to the
    CPU legs: torchrun sets OMP_NUM_THREADS=1 for its workers, which would
    otherwise leave the N > 1 reference arm on one core."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _cpu_call(streamed, family, op, herm, a, x, y, threads=0):
    if family == "symv":
        streamed.symv(op, 1.0, a, x, 0.0, y, hermitian=herm, nthreads=threads)
    else:
        streamed.gemv(op, 1.0, a, x, 0.0, y, nthreads=threads)


def cpu_baseline(seconds: float, opname: str, n: int, n_work: int, max_calls: int | None = None):
    """The oracle (C restatement of the reference's naive_gemv /
    naive_symv_hemv, all host threads) on the --op workload at order n; GB/s
    on the same algorithmic bytes."""
    from oracle import streamed  # CPU baseline leg only

    tag, family, op, herm, a, x, y, nbytes = _cpu_problem(opname, n)
    threads = host_threads()
    _cpu_call(streamed, family, op, herm, a, x, y, threads)  # warm
    calls, t0 = 0, time.perf_counter()
    while True:
        _cpu_call(streamed, family, op, herm, a, x, y, threads)
        calls += 1
        el = time.perf_counter() - t0
        if el >= seconds or (max_calls and calls >= max_calls):
            break
    gbs = nbytes * calls / el / 1e9
    return {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port", "cpu_model": cpu_model(),
            "sample": f"oracle/streamed.c {opname} ({op}) N={n} " + ("(the whole workload" if n == n_work else
                      f"(bounded sample of N={n_work}") + f", host matrix, wide accumulation), {calls} calls in "
                      f"{el:.1f} s, {threads} threads"}


def metric_name(opname: str) -> str:
    tag, family, op, herm = OPS[opname]
    label = {"symv": "SYMV" if not herm else "HEMV", "gemv": "GEMV"}[family]
    if opname == "dsymv":
        return "achieved HBM GB/s (DSYMV lower, algorithmic bytes)"
    return f"achieved HBM GB/s ({tag.upper()}{label}{'' if family == 'symv' else '-' + op.upper()}, algorithmic bytes)"


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port), rank 0 only,
    on the same workload (the whole operand when host RAM holds it)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import streamed

    northstar = args.op is None
    opname = args.op or "dsymv"
    if northstar:
        n_work = args.n or NS_N
    else:
        n_work = args.n or (32768 if OPS[opname][1] == "symv" else 16384)
    n = cpu_symv_n(n_work) if (northstar or n_work > CPU_SAMPLE_N and OPS[opname][1] == "symv") else min(
        n_work, CPU_SAMPLE_N)
    tag, family, op, herm, a, x, y, nbytes = _cpu_problem(opname, n)
    threads = host_threads()
    for _ in range(args.warmup):
        _cpu_call(streamed, family, op, herm, a, x, y, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _cpu_call(streamed, family, op, herm, a, x, y, threads)
    el = time.perf_counter() - t0
    gbs = nbytes * args.steps / el / 1e9
    whole = n == n_work
    sample = (f"oracle/streamed.c (C restatement of blockmv naive_symv_hemv / naive_gemv) {opname} N={n}, host "
              f"matrix, {threads} threads ({cpu_model()}); " +
              ("the whole workload" if whole else f"bounded sample of N={n_work}") +
              (" computed on one host (the reference's mgpu path is a host loop over the same column blocks, "
               "multidevice.py:183-284)" if northstar else ""))
    if northstar:
        workload, metric, scaling = NS_WORKLOAD.replace("G GPUs", f"{args.gpus} GPU(s)"), NS_METRIC, "strong"
    else:
        workload = ("DSYMV lower N=32768 (BASELINE configs[1])" if opname == "dsymv" and n_work == 32768
                    else "DGEMV non-transposed N=4096 (BASELINE configs[0])" if opname == "dgemv" and n_work == 4096
                    else f"{opname} m={n_work} n={n_work}")
        metric, scaling = metric_name(opname), "weak"
    line = {
        "impl": "reference", "metric": metric, "value": round(gbs, 3),
        "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(el / args.steps * 1e3, 4), "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": DTYPE_NAME[tag],
        "data": "synthetic U(-1,1)",
        "config": {"workload": workload, "cpu_sample_n": n, "op": opname, "n": n_work},
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- helpers
class Cublas:
    """cuBLAS (the torch wheel's libcublas) on the same device buffers: the
    library comparator BASELINE configs[1] names ("vs ... cuBLAS dsymv")."""

    def __init__(self):
        import ctypes
        import glob

        import torch

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

    def dsymv(self, uplo, n, A, ld, x, y, stream) -> bool:
        import ctypes

        if self.lib is None:
            return False
        self.lib.cublasSetStream_v2(self.h, ctypes.c_void_p(stream))
        one, zero = ctypes.c_double(1.0), ctypes.c_double(0.0)
        vp = ctypes.c_void_p
        rc = self.lib.cublasDsymv_v2(self.h, 0 if uplo == "l" else 1, n, ctypes.byref(one), vp(A), ld, vp(x), 1,
                                     ctypes.byref(zero), vp(y), 1)
        return rc == 0

    def close(self):
        if self.lib is not None:
            self.lib.cublasDestroy_v2(self.h)


def event_time(step, steps, dev, stream=None, barrier=None):
    """ms per step over `steps` calls, CUDA events on the launching stream,
    synchronize (and barrier) on both sides."""
    import torch

    stream = stream or torch.cuda.current_stream(dev)
    torch.cuda.synchronize(dev)
    if barrier:
        barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        step(i)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if barrier:
        barrier()
    return e0.elapsed_time(e1) / steps


def kernel_time(step, steps, dev):
    """Average duration of the library's dominant (streaming) kernel: the
    library's own CUDA-event brackets around each streaming launch, in a
    separate pass (the extra event records would break the PDL overlap of
    the timed region)."""
    import torch

    from paper_1410_1726_b200 import _lib

    _lib.timing_read()  # drop stale brackets
    _lib.timing_enable(True)
    for i in range(steps):
        step(i)
    torch.cuda.synchronize(dev)
    _lib.timing_enable(False)
    ms, k = _lib.timing_read()
    return ms / max(k, 1), k


# ------------------------------------------------------------- GPU arm
def bench_single(args, dev, rank, opname=None, n=None, m=None, steps=None, warmup=None, cublas=False,
                 sample_clocks=True):
    import torch

    from paper_1410_1726_b200 import _lib
    from paper_1410_1726_b200.core import precision

    opname = opname or args.op
    steps = steps or args.steps
    warmup = warmup if warmup is not None else args.warmup
    tag, family, op, herm = OPS[opname]
    p = precision(tag)
    n = n or args.n or (32768 if family == "symv" else 16384)
    m = n if family == "symv" else (m or args.m or n)
    lib = _lib.load()
    torch.manual_seed(0)
    ld = -(-m // 32) * 32
    # column-major A: a (n, ld) row-major tensor whose row j is column j
    A = torch.empty(n, ld, dtype=p.torch_dtype, device=dev)
    (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1)
    # operands smaller than 8x the 126 MB L2 rotate over copies of A (>= 1
    # GiB together), so every step streams its matrix from HBM even with
    # consecutive steps overlapping (programmatic dependent launch)
    ncopies = max(1, min(16, -(-(1 << 30) // A.numel() // p.element_bytes)))
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
    for i in range(warmup):
        step(i)
    torch.cuda.synchronize(dev)
    plan = _lib.last_plan()
    clock = ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) if sample_clocks else None
    if clock:
        clock.start()
        time.sleep(0.3)
    # warm the clocks up to the sampler's first reading, then time exactly K steps
    for i in range(warmup):
        step(i)
    l0 = _lib.launch_count()
    ms_step = event_time(step, steps, dev, stream)
    launches = _lib.launch_count() - l0
    clocks = clock.stop() if clock else None
    if launches == steps:
        # one library kernel per step (e.g. the row-owning GEMV-N): its
        # average launch duration is the timed region's event time over its
        # launches; per-launch brackets would add an event record between
        # back-to-back ~25 us kernels and overstate each by ~10 %
        kern_avg, kern_n = ms_step, launches
        ktiming = "one library kernel per step: timed-region CUDA events / launches"
    else:
        kern_avg, kern_n = kernel_time(step, min(steps, 50), dev)
        ktiming = "library CUDA-event brackets around each streaming launch (separate pass)"
    gbs = nbytes / (ms_step * 1e-3) / 1e9
    res = dict(tag=tag, family=family, op=op, opname=opname, m=m, n=n, ld=ld, nbytes=nbytes, nflops=nflops,
               ms_step=ms_step, gbs=gbs, kern_avg_ms=kern_avg, kern_launches=kern_n, launches=launches, plan=plan,
               clocks=clocks, ncopies=ncopies, kern_timing=ktiming)
    if cublas and family == "symv" and tag == "d":
        cub = Cublas()
        y2 = torch.empty_like(y)

        def theirs(i=0):
            assert cub.dsymv(op, n, As[i % ncopies].data_ptr(), ld, x.data_ptr(), y2.data_ptr(), sh)

        if cub.lib is not None:
            for i in range(warmup):
                theirs(i)
            cms = event_time(theirs, steps, dev, stream)
            step(0)
            theirs(0)
            torch.cuda.synchronize(dev)
            res["cublas"] = {"routine": "cublasDsymv_v2 (libcublas 12.9, CUBLAS_FILL_MODE_LOWER)",
                             "value": round(nbytes / (cms * 1e-3) / 1e9, 2), "unit": "GB/s",
                             "ms_per_step": round(cms, 5), "ours_over_cublas": round(cms / ms_step, 3),
                             "max_rel_diff": float(((y - y2).abs().max() / y2.abs().max()).item())}
        cub.close()
    # end to end through the public API with host (pinned) buffers
    if not args.no_e2e and args.e2e_steps > 0:
        res["e2e"] = e2e_single(args, As, x, y, tag, family, op, herm, m, n, ld, dev, nbytes)
    del As, A
    return res


def e2e_single(args, As, x, y, tag, family, op, herm, m, n, ld, dev, nbytes):
    """End to end through the public API (paper_1410_1726_b200.symv_hemv /
    gemv), as an iterative solver calls it: the matrix stays resident in HBM
    (uploaded once, like model weights), and every step copies that step's
    input x from pinned host memory to the device (y too when beta != 0; the
    bench uses beta = 0, so y is never read), runs the kernels and reads y
    back to the host.  A second figure re-uploads the referenced part of A
    every step as well (host-resident matrix), for transparency."""
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

        # warm-up holds three results at once, so the page-locked result
        # pool has the buffers the steady state rotates through (a first
        # allocation can take ~10 ms)
        warm = [step(i) for i in range(3)]
        del warm
        torch.cuda.synchronize(dev)
        ts = []
        t0 = time.perf_counter()
        for i in range(steps):
            t1 = time.perf_counter()
            out = step(i)
            ts.append(time.perf_counter() - t1)
        torch.cuda.synchronize(dev)
        run.per_step = sorted(ts)
        return (time.perf_counter() - t0) / steps, out

    # resident matrix (rotating over the same copies as the device-timed
    # steps): the headline end-to-end figure
    A = As[0]
    nsteps = max(args.e2e_steps, 50)
    el, out = run([kb.MatrixView(a.reshape(-1), m, n, ld, p) for a in As], nsteps)
    y_len = len(out)
    ps = run.per_step
    res = {"value": round(nbytes / el / 1e9, 3), "unit": "GB/s",
           "h2d_bytes_per_step": int(x_len * eb), "d2h_bytes_per_step": int(y_len * eb),
           "steps": nsteps, "ms_per_step": round(el * 1e3, 4),
           "step_ms": {"min": round(ps[0] * 1e3, 4), "median": round(ps[len(ps) // 2] * 1e3, 4),
                       "max": round(ps[-1] * 1e3, 4)},
           "path": f"paper_1410_1726_b200.{'symv_hemv' if family == 'symv' else 'gemv'} with A resident in HBM "
                   "(uploaded once), x from pinned host numpy each step (beta = 0: y is not uploaded), "
                   "y returned as numpy"}
    # the same calls queued (gemv_async / symv_hemv_async on a CommandQueue,
    # the reference's queue contract): no host wait per call, so the copies,
    # kernels and result writes of consecutive steps pipeline; the queue
    # synchronises every 16 steps and every step's result is read on the host
    q = kb.CommandQueue()
    hxs = [torch.empty(x.numel(), dtype=x.dtype, pin_memory=True).copy_(x) for _ in range(16)]
    npxs = [h.numpy() for h in hxs]
    views = [kb.MatrixView(a.reshape(-1), m, n, ld, p) for a in As]

    def qstep(i):
        view = views[i % len(views)]
        if family == "symv":
            return kb.symv_hemv_async(op, 1.0, kb.HermitianView(view, op), npxs[i % 16], 0.0, npy, queue=q,
                                      hermitian=herm)
        return kb.gemv_async(op, 1.0, view, npxs[i % 16], 0.0, npy, queue=q)

    def qrun(steps):
        hs = []
        for i in range(steps):
            hs.append(qstep(i))
            if len(hs) == 16 or i == steps - 1:
                q.synchronize()
                for h in hs:
                    float(h.result().y_out[0])  # host read of the step's result
                hs = []

    # warm-up of three batches: while a batch's results are being read the
    # previous batch's are still referenced, so the page-locked result pool
    # needs two batches of buffers before the timed steps (a pinned
    # allocation inside them costs milliseconds)
    qrun(48)
    torch.cuda.synchronize(dev)
    qsteps = max(64, nsteps)
    t0 = time.perf_counter()
    qrun(qsteps)
    torch.cuda.synchronize(dev)
    elq = (time.perf_counter() - t0) / qsteps
    res["queued"] = {"value": round(nbytes / elq / 1e9, 3), "unit": "GB/s", "ms_per_step": round(elq * 1e3, 4),
                     "h2d_bytes_per_step": int(x_len * eb), "d2h_bytes_per_step": int(y_len * eb),
                     "steps": qsteps,
                     "path": f"paper_1410_1726_b200.{'symv_hemv_async' if family == 'symv' else 'gemv_async'} on a "
                             "CommandQueue: x from pinned host numpy each step, result written to page-locked host "
                             "memory and read on the host after queue.synchronize() every 16 steps"}
    if family == "symv" and n >= 16384:
        # host-resident matrix: the referenced part of A is uploaded every step too
        hA = torch.empty(A.numel(), dtype=A.dtype, pin_memory=True)
        hA.copy_(A.reshape(-1))
        el2, _ = run([kb.MatrixView(hA.numpy(), m, n, ld, p)], args.e2e_steps)
        blocks = [(b0, min(n, b0 + 256)) for b0 in range(0, n, 256)]
        h2d_a = sum((b1 - b0) * ((m - b0) if op == "l" else b1) for b0, b1 in blocks) * eb
        res["with_matrix_upload"] = {
            "value": round(nbytes / el2 / 1e9, 3), "unit": "GB/s", "ms_per_step": round(el2 * 1e3, 3),
            "h2d_bytes_per_step": int(h2d_a + x_len * eb), "d2h_bytes_per_step": int(y_len * eb),
            "steps": args.e2e_steps,
            "path": "same call with A in pinned host memory: the stored triangle crosses PCIe every step "
                    "(INTEGRATION.md: keep A resident)"}
        del hA
    return res


# ------------------------------------------------------------- mgpu arm
def my_triangle_bytes(n, nb, world, rank, eb, uplo="l"):
    """Stored-triangle bytes of rank's block columns (its kernel's share of
    the algorithmic bytes)."""
    tot = 0
    for j in range(rank, -(-n // nb), world):
        c0, c1 = j * nb, min(n, (j + 1) * nb)
        w = c1 - c0
        other = (n - c1) if uplo == "l" else c0
        tot += (w * (w + 1) // 2 + other * w) * eb
    return tot


def bench_mgpu(args, dev, rank, world, opname, n, nb, exchanges=("p2p", "nccl"), headline="p2p"):
    """mgpu SYMV/HEMV over the 1D block-column-cyclic layout, one process
    per GPU: this rank's panel, partial via the sm_100a kernels, exchange of
    y onto rank 0.  Times every exchange in `exchanges` plus the
    partial-only step (no exchange), all max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1410_1726_b200 import _lib
    from paper_1410_1726_b200.core import MatrixView, precision
    from paper_1410_1726_b200.dist import P2PExchange, combine, p2p_mv, panel_shape
    from paper_1410_1726_b200.multidevice import partial_mv

    tag, family, op, herm = OPS[opname]
    if family != "symv":
        raise SystemExit("mgpu bench covers symv/hemv")
    p = precision(tag)
    rows, lc, ld = panel_shape(n, n, nb, world, rank)
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    panel_t = torch.empty(max(lc, 1) * ld, dtype=p.torch_dtype, device=dev)
    (torch.view_as_real(panel_t) if p.is_complex else panel_t).uniform_(-1, 1, generator=g)
    panel = MatrixView(panel_t, n, lc, ld, p) if lc > 0 else None
    x = torch.empty(n, dtype=p.torch_dtype, device=dev)
    (torch.view_as_real(x) if p.is_complex else x).uniform_(-1, 1, generator=torch.Generator(device=dev).manual_seed(7))
    out = torch.empty(n, dtype=p.torch_dtype, device=dev)
    nbytes = alg_bytes(tag, "symv", n, n, op)
    my_bytes = my_triangle_bytes(n, nb, world, rank, p.element_bytes, op)

    cdev = dev if dist.get_backend() == "nccl" else torch.device("cpu")  # gloo: host tensors

    def gather_max(v):
        t = torch.tensor([v], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def gather_all(v):
        t = torch.zeros(world, dtype=torch.float64, device=cdev)
        t[rank] = v
        dist.all_reduce(t)
        return [round(a, 5) for a in t.tolist()]

    def partial_step(i=0):
        partial_mv(p, "s", op, n, n, 1.0, panel, x, out, world, rank, nb, herm)

    ex = None
    steps_fn = {}
    if "p2p" in exchanges:
        try:
            ex = P2PExchange(n, p.torch_dtype)
        except Exception as err:  # no IPC between these ranks
            print(f"p2p exchange unavailable ({err})", file=sys.stderr, flush=True)
        if ex is not None:
            steps_fn["p2p"] = lambda i=0: p2p_mv(p, "s", op, n, n, 1.0, panel, x, 0.0, None, nb, ex, hermitian=herm)
    if "nccl" in exchanges:
        def nccl_step(i=0):
            partial_step()
            combine(out, None, 0.0)
        steps_fn["nccl"] = nccl_step
    if not steps_fn:
        raise SystemExit("no exchange available: p2p failed and NCCL cannot run with ranks sharing a GPU")
    if headline not in steps_fn:
        headline = next(iter(steps_fn))

    res = {"tag": tag, "op": op, "opname": opname, "n": n, "nb": nb, "ld": ld, "nbytes": nbytes,
           "my_bytes": my_bytes, "exchange": {}, "headline": headline}
    for name in [headline] + [e for e in steps_fn if e != headline]:
        step = steps_fn[name]
        for i in range(args.warmup):
            step(i)
        clock = None
        if name == headline:
            clock = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
            clock.start()
            time.sleep(0.3)
            for i in range(args.warmup):
                step(i)
        l0 = _lib.launch_count()
        ms = event_time(step, args.steps, dev, barrier=dist.barrier)
        launches = _lib.launch_count() - l0
        ent = {"ms_per_step": round(gather_max(ms), 5), "per_rank_ms": gather_all(ms)}
        ent["value"] = round(nbytes / (ent["ms_per_step"] * 1e-3) / 1e9, 2)
        if name == headline:
            res["clocks"] = clock.stop()
            res["launches"] = int(sum(gather_all(launches)))
            res["plan"] = _lib.last_plan()
        res["exchange"][name] = ent
    # partial only (no exchange) and the streaming kernel alone, per rank
    for i in range(args.warmup):
        partial_step(i)
    pms = event_time(partial_step, args.steps, dev, barrier=dist.barrier)
    kms, kn = kernel_time(partial_step, min(args.steps, 30), dev)
    res["per_rank"] = {"partial_only_ms": gather_all(pms), "kernel_ms": gather_all(kms),
                       "kernel_bytes": [int(b) for b in gather_all(my_bytes)],
                       "kernel_gbs": [round(b / (k * 1e-3) / 1e9, 1) if k > 0 else None
                                      for b, k in zip(gather_all(my_bytes), gather_all(kms))]}
    for name, ent in res["exchange"].items():
        ent["exchange_cost_ms"] = round(ent["ms_per_step"] - max(res["per_rank"]["partial_only_ms"]), 5)
    res["kern_avg_ms"] = kms
    res["ms_step"] = res["exchange"][headline]["ms_per_step"]
    res["gbs"] = nbytes / (res["ms_step"] * 1e-3) / 1e9
    if not args.no_e2e and args.e2e_steps > 0:
        res["e2e"] = e2e_mgpu(args, panel, x, out, p, n, nb, world, rank, dev, op, herm, nbytes,
                              ex if headline == "p2p" else None)
    torch.cuda.synchronize(dev)
    dist.barrier()
    if ex is not None:
        ex.close()
    del panel, panel_t
    torch.cuda.empty_cache()
    return res


def e2e_mgpu(args, panel, x, out, p, n, nb, world, rank, dev, op, herm, nbytes, ex=None):
    """Per step on every rank: x from pinned host to HBM, the partial kernels
    on the resident panel, the exchange onto rank 0 (peer-memory slots, or
    an NCCL reduce), and on rank 0 the D2H read of y.  Max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1410_1726_b200.dist import combine, p2p_mv
    from paper_1410_1726_b200.multidevice import partial_mv

    eb = p.element_bytes
    hx = torch.empty(n, dtype=x.dtype, pin_memory=True)
    hx.copy_(x)
    hy = torch.empty(n, dtype=x.dtype, pin_memory=True)
    dx = torch.empty_like(x)

    def step():
        dx.copy_(hx, non_blocking=True)
        if ex is not None:
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
    el = torch.tensor([(time.perf_counter() - t0) / steps],
                      device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    el = el.item()
    how = ("partial written into rank 0's peer-memory slot, device-flag handshake, rank-order combine in rank 0's "
           "epilogue" if ex is not None else "NCCL reduce to rank 0")
    return {"value": round(nbytes / el / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": int(world * n * eb),
            "d2h_bytes_per_step": int(n * eb), "steps": steps, "ms_per_step": round(el * 1e3, 4),
            "path": f"per rank: x from pinned host (H2D), kblas_mv_mgpu_partial_p2p_async / _partial_async on the "
                    f"HBM-resident panel, {how}, D2H of y on rank 0; max over ranks"}


def free_hbm_all(dev):
    """Free HBM (bytes) on the tightest rank."""
    import torch
    import torch.distributed as dist

    torch.cuda.empty_cache()
    f = torch.tensor([float(torch.cuda.mem_get_info(dev)[0])], dtype=torch.float64)
    if dist.is_initialized():
        if dist.get_backend() == "nccl":
            f = f.to(dev)
        dist.all_reduce(f, op=dist.ReduceOp.MIN)
    return f.item()


def roofline_of(bytes_per_launch, kern_ms, hbm_peak, peak_src, kernel, traffic_key):
    achieved = bytes_per_launch / (kern_ms * 1e-3) / 1e9 if kern_ms > 0 else None
    return {"bound": "hbm", "achieved": round(achieved, 2) if achieved else None, "peak": hbm_peak, "unit": "GB/s",
            "frac": round(achieved / hbm_peak, 4) if achieved else None, "traffic": traffic_of(traffic_key),
            "peak_source": peak_src, "kernel": kernel, "kernel_avg_ms": round(kern_ms, 5),
            "spec_peak_gbs": SPEC_HBM_GBS, "bytes_per_launch": int(bytes_per_launch)}


def single_block(res, hbm_peak, peak_src, workload):
    """Summary of a single-GPU run as an extra block of the N=1 line."""
    out = {"workload": workload, "op": res["opname"], "m": res["m"], "n": res["n"], "ld": res["ld"],
           "value": round(res["gbs"], 2), "unit": "GB/s", "ms_per_step": round(res["ms_step"], 5),
           "pct_of_copy_peak": round(100 * res["gbs"] / hbm_peak, 2),
           "gflops": round(res["nflops"] / (res["ms_step"] * 1e-3) / 1e9, 2),
           "roofline": dict(roofline_of(res["nbytes"], res["kern_avg_ms"], hbm_peak, peak_src,
                                        "kblas_" + res["plan"].split()[0] + "_kernel", f"{res['opname']}_{res['n']}"),
                            kernel_timing=res.get("kern_timing")),
           "gpu_launches": res["launches"], "plan": res["plan"],
           "l2": ("inputs > 126 MB L2 (A streamed from HBM every step), no flush" if res["ncopies"] == 1 else
                  f"{res['ncopies']} rotating copies of A (>= 1 GiB together, > 8x the L2)")}
    if res.get("clocks"):
        out["clocks"] = res["clocks"]
    for k in ("cublas", "e2e"):
        if k in res:
            out[k] = res[k]
    return out


def shared_gpus(world: int) -> bool:
    import torch

    return world > torch.cuda.device_count()


def free_port() -> str:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return str(port)


def run_northstar(args, dev, rank, world, hbm_peak, peak_src):
    """configs[4] at every N (strong scaling), plus the extra blocks."""
    import torch

    n, nb = args.n or NS_N, args.nb
    exchanges = ("p2p",) if shared_gpus(world) else ("p2p", "nccl")
    res = bench_mgpu(args, dev, rank, world, "dsymv", n, nb, exchanges)
    ex = res["exchange"]
    kern = max(res["per_rank"]["kernel_ms"])
    kr = res["per_rank"]["kernel_ms"].index(kern)
    line = None
    if rank == 0:
        line = {
            "metric": NS_METRIC,
            "value": round(res["gbs"], 2),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(res["ms_step"], 5),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic U(-1,1), generated on device per rank",
            "config": {"workload": NS_WORKLOAD.replace("G GPUs", f"{world} GPU(s)"), "op": "dsymv", "uplo": "l",
                       "n": n, "nb": nb, "ld": res["ld"], "alpha": 1.0, "beta": 0.0,
                       "exchange": "p2p (headline): partials stored into rank 0's HBM slots by the SYMV epilogue, "
                                   "rank-order sum there; nccl: partial kernels + NCCL reduce(sum) to rank 0",
                       "l2": "inputs >> 126 MB L2 (40 GB triangle, A streamed from HBM every step), no flush",
                       "parallelism": f"{world} GPU(s), one process each, 1D block-column-cyclic"},
            "pct_of_copy_peak": round(100 * res["gbs"] / (hbm_peak * world), 2),
            "gflops": round(alg_flops("d", "symv", n, n, "l") / (res["ms_step"] * 1e-3) / 1e9, 2),
            "roofline": roofline_of(res["per_rank"]["kernel_bytes"][kr], kern, hbm_peak, peak_src,
                                    "kblas_symv_kernel", f"mgpu_dsymv_{n}_G{world}"),
            "clocks": res["clocks"],
            "gpu_launches": res["launches"],
            "plan": res["plan"],
            "exchange": ex,
            "per_rank": res["per_rank"],
        }
        line["roofline"]["rank"] = kr
        line["e2e"] = res.get("e2e")
    if not args.no_extra:
        # ZHEMV N=100000 (configs[4]'s second routine): 160 GB at G=1
        from paper_1410_1726_b200.multidevice import local_col_count, local_ld

        need = max(local_col_count(n, nb, world, r) for r in range(world)) * local_ld(n) * 16
        if free_hbm_all(dev) > need + (6 << 30):
            zres = bench_mgpu(args, dev, rank, world, "zhemv", n, nb, exchanges)
            if rank == 0:
                zk = max(zres["per_rank"]["kernel_ms"])
                zr = zres["per_rank"]["kernel_ms"].index(zk)
                line["zhemv_100k"] = {
                    "workload": f"mgpu ZHEMV lower N={n}, nb={nb}, over {world} GPU(s) (BASELINE configs[4])",
                    "value": round(zres["gbs"], 2), "unit": "GB/s", "ms_per_step": round(zres["ms_step"], 5),
                    "exchange": zres["exchange"], "per_rank": zres["per_rank"], "plan": zres["plan"],
                    "roofline": roofline_of(zres["per_rank"]["kernel_bytes"][zr], zk, hbm_peak, peak_src,
                                            "kblas_symv_kernel", f"mgpu_zhemv_{n}_G{world}"),
                    "e2e": zres.get("e2e")}
        elif rank == 0:
            line["zhemv_100k"] = {"skipped": f"needs {need / 2**30:.0f} GiB of HBM per GPU"}
        if world == 1:
            r1 = bench_single(args, dev, rank, "dsymv", 32768, cublas=True, sample_clocks=False)
            line["configs1_dsymv_32768"] = single_block(r1, hbm_peak, peak_src,
                                                        "DSYMV lower N=32768 single B200 (BASELINE configs[1])")
            torch.cuda.empty_cache()
            r0 = bench_single(args, dev, rank, "dgemv", 4096, 4096, steps=max(args.steps, 200),
                              sample_clocks=False)
            line["configs0_dgemv_4096"] = single_block(r0, hbm_peak, peak_src,
                                                       "DGEMV non-transposed N=4096 (BASELINE configs[0])")
            torch.cuda.empty_cache()
    if rank == 0 and not args.no_cpu and world == 1:
        ncpu = cpu_symv_n(n)
        line["cpu_baseline"] = cpu_baseline(args.cpu_seconds, "dsymv", ncpu, n, max_calls=max(3, args.steps))
    return line


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
    # more ranks than GPUs (a functional run of the N>1 path on a 1-GPU box;
    # its timings are not scaling figures): ranks share devices round robin
    dev = torch.device("cuda", local % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)
    northstar = args.op is None
    mgpu = northstar or world > 1 or args.mgpu
    if mgpu:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if "MASTER_PORT" not in os.environ:
            os.environ["MASTER_PORT"] = free_port()
        if shared_gpus(world):
            # NCCL refuses two ranks on one device: gloo for the control
            # plane, and only the peer-memory exchange is timed
            dist.init_process_group("gloo", rank=rank, world_size=world)
        else:
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    hbm_peak, peak_src = measured_peaks()
    if northstar:
        line = run_northstar(args, dev, rank, world, hbm_peak, peak_src)
        if rank == 0:
            print(json.dumps(line), flush=True)
    elif mgpu:
        n = args.n or NS_N
        res = bench_mgpu(args, dev, rank, world, args.op, n, args.nb, exchanges=(args.reduce,),
                         headline=args.reduce)
        if rank == 0:
            kern = max(res["per_rank"]["kernel_ms"])
            kr = res["per_rank"]["kernel_ms"].index(kern)
            tag = res["tag"]
            line = {"metric": f"mgpu {metric_name(args.op)}", "value": round(res["gbs"], 2), "unit": "GB/s",
                    "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                    "ms_per_step": round(res["ms_step"], 5), "higher_is_better": True, "scaling": "strong",
                    "vs_baseline": None, "dtype": DTYPE_NAME[tag], "data": "synthetic U(-1,1), generated on device",
                    "config": {"workload": f"mgpu {args.op} N={n} nb={args.nb} over {world} GPU(s), {args.reduce}",
                               "n": n, "nb": args.nb},
                    "roofline": roofline_of(res["per_rank"]["kernel_bytes"][kr], kern, hbm_peak, peak_src,
                                            "kblas_symv_kernel", f"mgpu_{args.op}_{n}_G{world}"),
                    "clocks": res["clocks"], "gpu_launches": res["launches"], "plan": res["plan"],
                    "exchange": res["exchange"], "per_rank": res["per_rank"], "e2e": res.get("e2e")}
            print(json.dumps(line), flush=True)
    else:
        res = bench_single(args, dev, rank, cublas=True)
        if rank == 0:
            tag, opname = res["tag"], args.op
            if opname == "dsymv" and res["n"] == 32768:
                workload = "DSYMV lower N=32768 (BASELINE configs[1])"
            elif opname == "dgemv" and res["n"] == 4096 and res["m"] == 4096:
                workload = "DGEMV non-transposed N=4096 (BASELINE configs[0])"
            else:
                workload = f"{opname} m={res['m']} n={res['n']}"
            blk = single_block(res, hbm_peak, peak_src, workload)
            line = {"metric": metric_name(opname), "value": blk["value"], "unit": "GB/s", "n_gpus": world,
                    "steps": args.steps, "warmup": args.warmup, "ms_per_step": blk["ms_per_step"],
                    "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": DTYPE_NAME[tag],
                    "data": "synthetic U(-1,1), generated on device",
                    "config": {"workload": workload, "op": opname, "m": res["m"], "n": res["n"], "ld": res["ld"],
                               "uplo_or_trans": res["op"], "alpha": 1.0, "beta": 0.0, "l2": blk["l2"],
                               "parallelism": "1 GPU"}}
            for k in ("pct_of_copy_peak", "gflops", "roofline", "clocks", "gpu_launches", "plan", "cublas", "e2e"):
                if k in blk:
                    line[k] = blk[k]
            if not args.no_cpu:
                n_work = res["n"]
                ncpu = min(n_work, CPU_SAMPLE_N)
                line["cpu_baseline"] = cpu_baseline(args.cpu_seconds, opname, ncpu, n_work)
            print(json.dumps(line), flush=True)
    if mgpu:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
