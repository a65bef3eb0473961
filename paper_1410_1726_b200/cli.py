"""`python -m paper_1410_1726_b200 run ...`: run one kernel on the B200 and
report it in the reference's `blockmv run` schema (cli.py:64-93, 96-233),
with the Kepler cost-model columns replaced by measured ones.

    python -m paper_1410_1726_b200 run --kernel symv --prec d --n 32768 --beta 0

Inputs follow the reference CLI exactly (cli.py:52-57, 100-125): one
``numpy.random.default_rng(seed)`` fills the parent (m+row_off) x
(n+col_off) matrix (ld padded to 32 elements), then x, then y, with
U(-1, 1) entries (complex: independent real and imaginary parts); the
Hermitian diagonal is made real.  So a row here and a row of the
reference's `blockmv run` describe the same problem.

Columns: the reference's counters (bytes_read ... scal_invocations, SURVEY
Appendix B: the algorithmic figures, not the 128-B segment model), then
measured_seconds (CUDA events, mean over --reps calls on HBM-resident
operands after --warmup calls), measured_gflops, achieved_gbs
(algorithmic bytes, roofline.py), the copy peak and the fraction of it,
and the verification columns.  `--devices G` adds one row per GPU as the
reference does (scope device-g).

Verification (the reference's `run` does the same against its naive
oracle, cli.py:163-178) is a column-panel product in wide precision
(f64 / c128) on the host, computed here only to check the GPU result; the
result itself always comes from the sm_100a kernels.  It is on by default
up to --verify-max (default 16384) and skipped above unless --verify.
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys

import numpy as np

RUN_CSV_HEADER = [
    "scope", "kernel", "precision", "m", "n", "nb", "q", "y", "row_off", "col_off", "devices",
    "bytes_read", "bytes_written", "transactions", "matrix_transactions", "flops", "tb_count",
    "atomic_adds", "reduction_events", "scal_invocations",
    "measured_seconds", "measured_gflops", "achieved_gbs", "copy_peak_gbs", "pct_copy_peak",
    "max_abs_error", "error_bound", "verified", "plan",
]

KERNEL_CHOICES = ("gemv", "gemv-t", "gemv-c", "symv", "hemv")
FALLBACK_COPY_PEAK_GBS = 6650.0  # B200_PROFILING.md fallback when no measured peak is available


def copy_peak() -> tuple[float, str]:
    """Measured HBM copy peak: $KBLAS_COPY_PEAK_GBS, else MEASURED_PEAKS.json
    in the working directory or the repo root, else the pool fallback."""
    env = os.environ.get("KBLAS_COPY_PEAK_GBS")
    if env:
        return float(env), "env"
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for d in (os.getcwd(), here):
        try:
            with open(os.path.join(d, "MEASURED_PEAKS.json")) as fh:
                return float(json.load(fh)["hbm_gbs"]), "measured"
        except (OSError, KeyError, ValueError):
            continue
    return FALLBACK_COPY_PEAK_GBS, "fallback"


def _fill(rng, shape, prec):
    """cli.py:52-57."""
    if prec.is_complex:
        re = rng.uniform(-1, 1, size=shape)
        im = rng.uniform(-1, 1, size=shape)
        return (re + 1j * im).astype(prec.dtype)
    return rng.uniform(-1, 1, size=shape).astype(prec.dtype)


def _wide(a):
    return a.astype(np.complex128 if np.iscomplexobj(a) else np.float64)


def check_gemv(trans, alpha, a, x, beta, y, eps, panel=1024):
    """max |y_gpu - y_ref| and the reference bound for a GEMV, column panels in
    wide precision: returns (y_ref, bound)."""
    m, n = a.shape
    xw, yw = _wide(x), _wide(y)
    if trans == "n":
        acc, rowabs = np.zeros(m, dtype=xw.dtype), np.zeros(m)
    else:
        acc, rowabs = np.zeros(n, dtype=xw.dtype), np.zeros(n)
    for j0 in range(0, n, panel):
        j1 = min(n, j0 + panel)
        blk = _wide(a[:, j0:j1])
        if trans == "n":
            acc = acc + blk @ xw[j0:j1]
            rowabs += np.abs(blk).sum(axis=1)
        else:
            op = blk.conj().T if trans == "c" else blk.T
            acc[j0:j1] = op @ xw
            rowabs[j0:j1] = np.abs(blk).sum(axis=0)
    want = alpha * acc + beta * yw
    bound = 50 * eps * (abs(alpha) * rowabs.max() * np.abs(xw).max() + abs(beta) * np.abs(yw).max())
    return want, bound


def check_symv(uplo, hermitian, alpha, a, x, beta, y, eps, panel=1024):
    """Same for SYMV/HEMV from the stored triangle of a (d x d): the panel is
    mirrored on the fly (conjugated for Hermitian, diagonal real)."""
    d = a.shape[0]
    xw, yw = _wide(x), _wide(y)
    acc, rowabs = np.zeros(d, dtype=xw.dtype), np.zeros(d)
    for j0 in range(0, d, panel):
        j1 = min(d, j0 + panel)
        r0, r1 = (j0, d) if uplo == "l" else (0, j1)
        blk = _wide(a[r0:r1, j0:j1])
        rows = np.arange(r0, r1)[:, None]
        cols = np.arange(j0, j1)[None, :]
        stored = rows >= cols if uplo == "l" else rows <= cols
        strict = rows > cols if uplo == "l" else rows < cols
        s = np.where(stored, blk, 0)
        if hermitian:
            diag = rows == cols
            s = np.where(diag, s.real, s)
        t = np.where(strict, blk, 0)
        tt = t.conj().T if hermitian else t.T
        acc[r0:r1] += s @ xw[j0:j1]
        acc[j0:j1] += tt @ xw[r0:r1]
        rowabs[r0:r1] += np.abs(s).sum(axis=1)
        rowabs[j0:j1] += np.abs(t).sum(axis=0)
    want = alpha * acc + beta * yw
    bound = 50 * eps * (abs(alpha) * rowabs.max() * np.abs(xw).max() + abs(beta) * np.abs(yw).max())
    return want, bound


def cmd_run(args) -> int:
    import torch

    from . import _lib, roofline
    from .core import HermitianView, make_padded_view, precision
    from .kernels import gemv, symv_hemv
    from .multidevice import distribute, gemv_mgpu, symv_hemv_mgpu
    from .offset import OffsetRequest, gemv_offset, symv_hemv_offset
    from .partition import KernelConfig

    prec = precision(args.prec)
    cfg = KernelConfig(block_size=args.nb, thread_cols=args.q, coop_tbs=args.y)
    symmetric = args.kernel in ("symv", "hemv")
    herm = args.kernel == "hemv"
    if herm and not prec.is_complex:
        print("error: hemv needs a complex precision (c or z)", file=sys.stderr)
        return 2
    n = args.n
    if n <= 0 or (args.m is not None and args.m <= 0):
        print("error: --m and --n must be positive", file=sys.stderr)
        return 2
    m = args.m if (args.m is not None and not symmetric) else n
    if symmetric and args.col_off not in (0, args.row_off):
        print("error: symmetric offsets must be diagonal (equal row/col)", file=sys.stderr)
        return 2
    if args.devices > 1 and (args.row_off or args.col_off):
        print("error: --devices cannot be combined with offsets", file=sys.stderr)
        return 2
    row_off, col_off = args.row_off, (args.row_off if symmetric else args.col_off)
    parent_m, parent_n = (n + row_off, n + row_off) if symmetric else (m + row_off, n + col_off)
    trans = {"gemv": "n", "gemv-t": "t", "gemv-c": "c"}.get(args.kernel)
    x_len, y_len = (n, m) if trans in (None, "n") else (m, n)

    dev = torch.device("cuda", torch.cuda.current_device())
    host_parent = make_padded_view(parent_m, parent_n, prec, pad_to=32, device="numpy")
    rng = np.random.default_rng(args.seed)
    host_parent.array()[:, :] = _fill(rng, (parent_m, parent_n), prec)
    if herm:
        ha = host_parent.array()
        idx = np.arange(min(parent_m, parent_n))
        ha[idx, idx] = ha[idx, idx].real
    x = _fill(rng, x_len, prec)
    y = _fill(rng, y_len, prec)
    alpha = prec.dtype.type(args.alpha)
    beta = prec.dtype.type(args.beta)

    parent = make_padded_view(parent_m, parent_n, prec, pad_to=32, device=dev)
    parent.data.copy_(torch.from_numpy(host_parent.data))
    sub = parent.submatrix(row_off, col_off, m, n)
    xd = torch.from_numpy(x).to(dev)
    yd = torch.from_numpy(y).to(dev)

    dist = distribute(parent, args.nb, args.devices) if args.devices > 1 else None

    def call():
        if dist is not None:
            if symmetric:
                return symv_hemv_mgpu(args.uplo, alpha, dist, xd, beta, yd, cfg, hermitian=herm)
            return gemv_mgpu(trans, alpha, dist, xd, beta, yd, cfg)
        if row_off or col_off:
            if symmetric:
                return symv_hemv_offset(args.uplo, alpha, HermitianView(base=parent, uplo=args.uplo), row_off, n,
                                        xd, beta, yd, cfg, hermitian=herm), []
            req = OffsetRequest(parent=parent, row_off=row_off, col_off=col_off, sub_m=m, sub_n=n)
            return gemv_offset(trans, alpha, req, xd, beta, yd, cfg), []
        if symmetric:
            return symv_hemv(args.uplo, alpha, HermitianView(base=sub, uplo=args.uplo), xd, beta, yd, cfg,
                             hermitian=herm), []
        return gemv(trans, alpha, sub, xd, beta, yd, cfg), []

    rep, per_device = call()
    for _ in range(args.warmup):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    seconds = e0.elapsed_time(e1) / 1e3 / max(args.reps, 1)

    nbytes = roofline.symv_bytes(prec, n) if symmetric else roofline.gemv_bytes(prec, m, n, trans)
    nflops = roofline.symv_flops(prec, n) if symmetric else roofline.gemv_flops(prec, m, n, trans)
    peak, _src = copy_peak()
    gbs = nbytes / seconds / 1e9

    verified, err_s, bound_s = "skipped", "", ""
    if args.verify or (args.verify is None and max(m, n) <= args.verify_max):
        got = rep.y_out.cpu().numpy()
        a_host = host_parent.array()[row_off:row_off + (n if symmetric else m), col_off:col_off + n]
        if symmetric:
            want, bound = check_symv(args.uplo, herm, alpha, a_host, x, beta, y, prec.eps)
        else:
            want, bound = check_gemv(trans, alpha, a_host, x, beta, y, prec.eps)
        err = float(np.max(np.abs(got.astype(want.dtype) - want))) if got.size else 0.0
        ok = err <= max(bound, 10 * prec.eps)
        verified, err_s, bound_s = ("pass" if ok else "FAIL"), f"{err:.3e}", f"{bound:.3e}"

    def row(scope, r, timed):
        return [
            scope, args.kernel, prec.tag, m, n, args.nb, args.q, args.y, row_off, col_off, args.devices,
            r.bytes_read, r.bytes_written, r.transactions, r.matrix_transactions, r.flops, r.tb_count,
            r.atomic_adds, r.reduction_events, r.scal_invocations,
            f"{seconds:.6e}" if timed else "", f"{nflops / seconds / 1e9:.4f}" if timed else "",
            f"{gbs:.2f}" if timed else "", f"{peak:.1f}", f"{gbs / peak:.4f}" if timed else "",
            err_s if timed else "", bound_s if timed else "", verified if timed else "", r.plan,
        ]

    fh = open(args.csv, "w", newline="") if args.csv and args.csv != "-" else sys.stdout
    try:
        w = csv.writer(fh)
        w.writerow(RUN_CSV_HEADER)
        w.writerow(row("merged", rep, True))
        for g, r in enumerate(per_device):
            w.writerow(row(f"device-{g}", r, False))
    finally:
        if fh is not sys.stdout:
            fh.close()
    if verified == "FAIL":
        print(f"verification FAILED: error {err_s} exceeds bound {bound_s}", file=sys.stderr)
        return 1
    _lib.load()
    return 0


def cmd_tune(args) -> int:
    """Measured coarse/fine search (reference cli.py:295-331): CSV of every
    timed point, the winners on stderr, optionally applied and saved as a
    tuning table (--save; load it with $KBLAS_TUNING_FILE)."""
    from . import tuner
    from .core import precision

    try:
        sizes = [int(s) for s in args.sizes.split(",") if s]
        if not sizes or min(sizes) <= 0:
            raise ValueError("--sizes needs positive orders")
        prec = precision(args.prec)
        tuner._check_kernel(args.kernel, prec)
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    import torch

    if not torch.cuda.is_available():
        print("error: tune needs a CUDA device (the tuner times the sm_100a kernels)", file=sys.stderr)
        return 2
    coarse, fine = tuner.tune(args.kernel, args.prec, sizes, uplo=args.uplo, reps=args.reps,
                              min_gain=args.min_gain)
    fh = open(args.csv, "w", newline="") if args.csv else sys.stdout
    try:
        tuner.write_sweep_csv(coarse.points + fine.points, fh)
    finally:
        if fh is not sys.stdout:
            fh.close()
    print(f"coarse winner: {coarse.winner.label()}; fine recommendation: {fine.recommended.label()}",
          file=sys.stderr)
    for size in sorted(fine.per_size):
        print(f"  size {size}: {fine.per_size[size].label()}", file=sys.stderr)
    if args.save:
        # the file holds this run's ranges (and, with --merge, the file's
        # earlier ranges for other kernels), never the library's built-in table
        old = tuner.read(args.save) if args.merge and os.path.exists(args.save) else []
        entries = tuner.merge_entries(old, fine)
        tuner.apply(fine)
        tuner.save(args.save, entries, device=torch.cuda.get_device_name())
        print(f"saved {len(entries)} tuned range(s) to {args.save}", file=sys.stderr)
    return 0


def cmd_roofline(args) -> int:
    """Intensity / bandwidth-bound table (reference cli.py:236-248), with
    the B200's measured copy bandwidth as the bound."""
    from . import roofline

    peak, source = copy_peak()
    fh = open(args.csv, "w", newline="") if args.csv else sys.stdout
    try:
        roofline.write_intensity_csv(fh, peak, source, args.sample_n)
    finally:
        if fh is not sys.stdout:
            fh.close()
    return 0


OFFSET_SCAN_HEADER = ["offset", "matrix_bytes", "measured_seconds", "achieved_gbs", "inflation"]


def cmd_offset_scan(args) -> int:
    """Measured counterpart of the reference's transaction-inflation scan
    (cli.py:251-292): the standard kernel on an n x n window at every row
    offset 0..max_off of one parent matrix, timed on the GPU; inflation is
    the time relative to offset 0 (the reference's modelled segment count
    has no meaning for the realigned 256-bit loads)."""
    from .core import precision

    try:
        prec = precision(args.prec)
        if args.n < 1 or args.max_off < 0:
            raise ValueError("--n must be >= 1 and --max-off >= 0")
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    import torch

    if not torch.cuda.is_available():
        print("error: offset-scan needs a CUDA device (it times the sm_100a kernels)", file=sys.stderr)
        return 2
    from . import _lib, roofline
    from .core import MatrixView

    dev = torch.device("cuda", torch.cuda.current_device())
    n, mo = args.n, args.max_off
    ld = -(-(n + mo) // 32) * 32
    base = torch.empty(ld * n, dtype=prec.torch_dtype, device=dev)
    (torch.view_as_real(base) if prec.is_complex else base).uniform_(-1, 1)
    parent = MatrixView(base, n + mo, n, ld, prec)
    x = torch.ones(n, dtype=prec.torch_dtype, device=dev)
    y = torch.empty(n, dtype=prec.torch_dtype, device=dev)
    trans = "n" if args.kernel == "gemv" else "t"
    f = getattr(_lib.load(), f"kblas_{prec.tag}gemv_async")
    one, zero = _lib.scalar(prec.tag, 1.0), _lib.scalar(prec.tag, 0.0)
    st = torch.cuda.current_stream(dev).cuda_stream
    nbytes = roofline.gemv_bytes(prec, n, n, trans)
    rows, t0 = [], None
    for off in range(mo + 1):
        sub = parent.submatrix(off, 0, n, n)
        ptr = base.data_ptr() + sub.linear_index(0, 0) * prec.element_bytes

        def call():
            _lib.check(f(trans.encode(), n, n, one, ptr, ld, x.data_ptr(), 1, zero, y.data_ptr(), 1, st),
                       "offset-scan")

        for _ in range(args.warmup):
            call()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            call()
        e1.record()
        torch.cuda.synchronize(dev)
        sec = e0.elapsed_time(e1) / 1e3 / args.reps
        t0 = sec if t0 is None else t0
        rows.append((off, nbytes, sec, nbytes / sec / 1e9, sec / t0))
    fh = open(args.csv, "w", newline="") if args.csv else sys.stdout
    try:
        w = csv.writer(fh)
        w.writerow(OFFSET_SCAN_HEADER)
        for off, b, sec, gbs, infl in rows:
            w.writerow([off, b, f"{sec:.9f}", f"{gbs:.1f}", f"{infl:.6f}"])
    finally:
        if fh is not sys.stdout:
            fh.close()
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="python -m paper_1410_1726_b200",
        description="Run B200 matrix-vector kernels and report measured throughput (blockmv run schema).")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("run", help="run one kernel on the GPU, time it and verify it")
    p.add_argument("--kernel", choices=KERNEL_CHOICES, required=True)
    p.add_argument("--prec", choices="sdcz", default="d")
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--m", type=int, default=None, help="rows (general kernels; defaults to n)")
    p.add_argument("--nb", type=int, default=64, help="KernelConfig block size; mgpu distribution width")
    p.add_argument("--q", type=int, default=4)
    p.add_argument("--y", type=int, default=1)
    p.add_argument("--uplo", choices=("l", "u"), default="l")
    p.add_argument("--alpha", type=float, default=1.0)
    p.add_argument("--beta", type=float, default=1.0)
    p.add_argument("--row-off", type=int, default=0)
    p.add_argument("--col-off", type=int, default=0)
    p.add_argument("--devices", type=int, default=1)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--reps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--verify", dest="verify", action="store_true", default=None,
                   help="verify against the wide-precision host product at any size")
    p.add_argument("--no-verify", dest="verify", action="store_false")
    p.add_argument("--verify-max", type=int, default=16384)
    p.add_argument("--csv", help="write the report here instead of stdout")
    p.set_defaults(func=cmd_run)

    p = sub.add_parser("roofline", help="emit the intensity / bandwidth-bound table for the B200")
    p.add_argument("--sample-n", type=int, default=1_000_000)
    p.add_argument("--csv", help="write the table here instead of stdout")
    p.set_defaults(func=cmd_roofline)

    p = sub.add_parser("offset-scan", help="measured time versus row offset (realignment check)")
    p.add_argument("--kernel", choices=("gemv", "gemv-t"), default="gemv")
    p.add_argument("--prec", choices="sdcz", default="s")
    p.add_argument("--n", type=int, default=4096)
    p.add_argument("--max-off", type=int, default=64)
    p.add_argument("--reps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--csv", help="write the scan here instead of stdout")
    p.set_defaults(func=cmd_offset_scan)

    p = sub.add_parser("tune", help="measured coarse/fine configuration search on the GPU")
    p.add_argument("--kernel", choices=KERNEL_CHOICES, required=True)
    p.add_argument("--prec", choices="sdcz", default="d")
    p.add_argument("--sizes", default="1024,2048,4096,8192")
    p.add_argument("--uplo", choices=("l", "u"), default="l")
    p.add_argument("--reps", type=int, default=20)
    p.add_argument("--min-gain", type=float, default=0.01,
                   help="fraction a candidate must beat the built-in choice by")
    p.add_argument("--csv", help="write the sweep here instead of stdout")
    p.add_argument("--save", help="apply the result and save the tuning table (JSON) here")
    p.add_argument("--merge", action="store_true", help="keep the entries already in --save")
    p.set_defaults(func=cmd_tune)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    return args.func(args)
