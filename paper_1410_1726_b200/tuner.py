"""Empirical on-device tuner: the B200 replacement of the reference's
analytic coarse/fine tuner (reference tuner.py:1-9, 168-235; SURVEY §8f
rank 1, following the paper's coarse -> fine procedure).

The reference scores (block_size, thread_cols, coop_tbs) candidates with a
transaction-ledger cost model.  Here every candidate is run and timed on the
GPU through the product C entry points (kblas_<x>gemv_async,
kblas_<x>symv/hemv_async).  Each candidate is a row of the library's tuning
table (kblas_tune_set), so what the tuner measures is exactly what a
tuned call later runs.

Candidates are a TuneConfig (shape, form, waves):

* shape: the streaming kernel's geometry, the analogue of (block_size,
  thread_cols).  GEMV: 3 = 4 warps x 4 columns x 2 vectors, 2 CTAs/SM;
  4 = 16 x 4 x 1, 1 CTA/SM; 5 = 8 x 4 x 1, 2 CTAs/SM.  SYMV/HEMV: 100 = wide
  tiles (16 warps x 8 columns), 103 = narrow (8 x 4), 105 = mid (8 x 8,
  2 CTAs/SM).  0 (GEMV) / -1 (SYMV) = the built-in rule.
* form: how the work of one row block (GEMV-N) or column block (GEMV-T/C)
  is shared between CTAs, the analogue of coop_tbs.  GEMV-N: 0 stacked-rows
  stream-K, 1 split form with global partial slots, 2 split form reduced in
  a thread-block cluster, 3 row-owning CTAs (whose shape 10..17 selects
  the configuration).  GEMV-T/C: 0 stream-K, 1 column-owning CTAs.
  -1 = built-in rule.
* waves: split-form GEMV-N grid size in waves of the GPU (0 = default).

Stage one (coarse_tune) times every shape at the largest size with the form
left to the built-in rule.  It keeps the winner, breaking ties toward the
built-in choice.  Stage two (fine_tune) keeps that shape and scans the forms
per size; SYMV/HEMV has no form knob, so its fine stage scans the shapes per
size.  A candidate must beat the built-in choice by `min_gain`
(default 1 %) before it replaces it, so noise does not rewrite the defaults.
Every candidate's result is checked against the built-in choice's on the
same inputs.

`apply()` installs a fine result into the running library: each tuned size
covers the orders closest to it (geometric midpoints), and nothing outside
[min/sqrt2, max*sqrt2] changes.  `save()` / `load()` keep a table as JSON;
the library loads $KBLAS_TUNING_FILE (a path) on first use, if set.
"""

from __future__ import annotations

import csv
import ctypes
import json
import math
import os
from dataclasses import asdict, dataclass, field

from . import _lib
from .core import Precision, precision

KERNELS = ("gemv", "gemv-t", "gemv-c", "symv", "hemv")
GEMV_SHAPES = (5, 3, 4)
SYMV_SHAPES = (100, 103, 105)
GEMV_N_FORMS = (0, 1, 2)
ROWOWN_SHAPES = tuple(range(10, 18))  # GEMV-N form 3: row-owning configuration 0..7
GEMV_T_FORMS = (0, 1)
AUTO_GEMV, AUTO_SYMV = 0, -1


@dataclass(frozen=True)
class TuneConfig:
    """One candidate: a row of the library's tuning table (kblas_tune_set)."""

    shape: int
    form: int = -1
    waves: int = 0

    @property
    def is_auto(self) -> bool:
        return self.shape in (AUTO_GEMV, AUTO_SYMV) and self.form == -1 and self.waves == 0

    def label(self) -> str:
        return f"shape={self.shape} form={self.form} waves={self.waves}"


def op_of(kernel: str, uplo: str = "l") -> str:
    """Table operation code for a tuner kernel name."""
    if kernel == "gemv":
        return "n"
    if kernel == "gemv-t":
        return "t"
    if kernel == "gemv-c":
        return "c"
    if kernel in ("symv", "hemv"):
        if uplo not in ("l", "u"):
            raise ValueError(f"uplo must be 'l' or 'u', got {uplo!r}")
        return uplo
    raise ValueError(f"unknown kernel {kernel!r}; expected one of {KERNELS}")


def _check_kernel(kernel: str, prec: Precision):
    op_of(kernel)
    if kernel == "hemv" and not prec.is_complex:
        raise ValueError("hemv needs a complex precision (c or z)")


def auto_config(kernel: str) -> TuneConfig:
    return TuneConfig(AUTO_SYMV if kernel in ("symv", "hemv") else AUTO_GEMV)


def enumerate_configs(kernel: str, stage: str = "coarse", shape: int | None = None) -> list[TuneConfig]:
    """Candidates of one stage (the built-in choice first).

    coarse: every shape, form left to the built-in rule (GEMV-T/C: the
    stream-K form, the only one the shape changes).  fine: the forms of
    `shape` (GEMV-N adds the split form at 2 waves); SYMV/HEMV: every shape.
    """
    op = op_of(kernel)
    out = [auto_config(kernel)]
    if op in ("l", "u"):
        out += [TuneConfig(s) for s in SYMV_SHAPES]
        return out
    if stage == "coarse":
        form = -1 if op == "n" else 0
        out += [TuneConfig(s, form) for s in GEMV_SHAPES]
        return out
    if stage != "fine":
        raise ValueError(f"stage must be 'coarse' or 'fine', got {stage!r}")
    base = AUTO_GEMV if shape is None else shape
    forms = GEMV_N_FORMS if op == "n" else GEMV_T_FORMS
    # the forms of the coarse shape and, when that is not the built-in
    # shape, of the built-in shape too (so runs whose coarse stages
    # disagree still time the same cells)
    for sh in dict.fromkeys((base, AUTO_GEMV)):
        out += [TuneConfig(sh, f) for f in forms]
        if op == "n":
            out.append(TuneConfig(sh, 1, 2))
    if op == "n":
        out += [TuneConfig(s, 3) for s in ROWOWN_SHAPES]
    if base != AUTO_GEMV:
        out.append(TuneConfig(base))
    return list(dict.fromkeys(out))


@dataclass(frozen=True)
class TunePoint:
    """Measured performance of one (kernel, precision, size, config) cell."""

    kernel: str
    precision: Precision
    size: int
    config: TuneConfig
    measured_gbs: float
    seconds: float
    rel_diff: float
    plan: str
    uplo: str = "l"


@dataclass(frozen=True)
class CoarseResult:
    winner: TuneConfig
    points: list[TunePoint]


@dataclass(frozen=True)
class FineResult:
    kernel: str
    precision: Precision
    uplo: str
    per_size: dict[int, TuneConfig]
    recommended: TuneConfig
    points: list[TunePoint] = field(default_factory=list)


# ---------------------------------------------------------------- table I/O
@dataclass(frozen=True)
class TableEntry:
    prec: str
    op: str
    n_lo: int
    n_hi: int
    shape: int
    form: int = -1
    waves: int = 0


def table() -> list[TableEntry]:
    """The library's current tuning table."""
    lib = _lib.load()
    out = []
    for i in range(int(lib.kblas_tune_count())):
        p, o = ctypes.create_string_buffer(1), ctypes.create_string_buffer(1)
        lo, hi = ctypes.c_longlong(), ctypes.c_longlong()
        sh, fo, wv = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        if lib.kblas_tune_get(i, p, o, ctypes.byref(lo), ctypes.byref(hi), ctypes.byref(sh), ctypes.byref(fo),
                              ctypes.byref(wv)) == 0:
            out.append(TableEntry(p.raw.decode(), o.raw.decode(), lo.value, hi.value, sh.value, fo.value, wv.value))
    return out


def set_entry(e: TableEntry):
    rc = _lib.load().kblas_tune_set(e.prec.encode(), e.op.encode(), int(e.n_lo), int(e.n_hi), int(e.shape),
                                    int(e.form), int(e.waves))
    _lib.check(rc, "kblas_tune_set", ["prec", "op", "n_lo", "n_hi", "shape", "form", "waves"])


def clear():
    """Empty the table: calls run on the built-in rules alone."""
    _lib.load().kblas_tune_clear()


def defaults() -> int:
    """Reinstall the measured table built into the library (BUILTIN_TABLE)."""
    return int(_lib.load().kblas_tune_defaults())


BUILTIN_TABLE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tuning", "b200.json")


def restore(entries: list[TableEntry]):
    clear()
    for e in entries:
        set_entry(e)


def save(path: str, entries: list[TableEntry] | None = None, device: str | None = None):
    entries = table() if entries is None else entries
    doc = {"format": "kblas-b200-tuning/1", "device": device, "entries": [asdict(e) for e in entries]}
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=1)
        fh.write("\n")


def read(path: str) -> list[TableEntry]:
    """The entries of a saved table (nothing is installed)."""
    with open(path) as fh:
        doc = json.load(fh)
    if doc.get("format") != "kblas-b200-tuning/1":
        raise ValueError(f"{path}: not a kblas-b200 tuning table")
    return [TableEntry(**e) for e in doc["entries"]]


def load(path: str, replace: bool = False) -> int:
    """Install a saved table; returns the number of entries added."""
    entries = read(path)
    if replace:
        clear()
    for e in entries:
        set_entry(e)
    return len(entries)


def merge_entries(old: list[TableEntry], result: FineResult) -> list[TableEntry]:
    """`old` with every entry of the result's (precision, op) replaced by
    the result's rows (a re-tune supersedes the earlier ranges)."""
    op = op_of("symv" if result.kernel in ("symv", "hemv") else result.kernel, result.uplo)
    kept = [e for e in old if (e.prec, e.op) != (result.precision.tag, op)]
    return kept + entries_for(result)


def entries_for(result: FineResult) -> list[TableEntry]:
    """Table rows for a fine result: each size covers the orders nearest to
    it on a log scale, within [min/sqrt2, max*sqrt2]; sizes whose winner is
    the built-in choice add nothing."""
    sizes = sorted(result.per_size)
    op = op_of("symv" if result.kernel in ("symv", "hemv") else result.kernel, result.uplo)
    out = []
    for i, n in enumerate(sizes):
        lo = math.ceil(n / math.sqrt(2)) if i == 0 else math.floor(math.sqrt(sizes[i - 1] * n)) + 1
        hi = math.floor(n * math.sqrt(2)) if i == len(sizes) - 1 else math.floor(math.sqrt(n * sizes[i + 1]))
        c = result.per_size[n]
        if c.is_auto:
            continue
        out.append(TableEntry(result.precision.tag, op, lo, hi, c.shape, c.form, c.waves))
    return out


def apply(result: FineResult) -> list[TableEntry]:
    """Install a fine result into the running library."""
    rows = entries_for(result)
    for e in rows:
        set_entry(e)
    return rows


# ----------------------------------------------------------------- measuring
class _Bench:
    """HBM-resident operands of one (kernel, precision, size), with enough
    rotating copies of A that consecutive calls do not hit L2."""

    L2_BYTES = 126 << 20

    def __init__(self, kernel: str, prec: Precision, n: int, uplo: str, seed: int = 0):
        import torch

        self.torch = torch
        self.kernel, self.prec, self.n, self.uplo = kernel, prec, n, uplo
        dev = torch.device("cuda", torch.cuda.current_device())
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        abytes = n * n * prec.element_bytes
        free = torch.cuda.mem_get_info(dev)[0]
        # rotating copies: together > 8x L2, so every call streams from HBM
        # (consecutive calls overlap under chained launches)
        copies = max(1, min(64, math.ceil(8 * self.L2_BYTES / max(1, abytes)), int(0.5 * free // max(1, abytes))))

        def rnd(*shape):
            t = torch.empty(*shape, dtype=prec.torch_dtype, device=dev)
            (torch.view_as_real(t) if prec.is_complex else t).uniform_(-1, 1, generator=g)
            return t

        self.As = [rnd(n, n) for _ in range(copies)]
        self.x = rnd(n)
        self.y = torch.zeros(n, dtype=prec.torch_dtype, device=dev)
        self.one, self.zero = _lib.scalar(prec.tag, 1.0), _lib.scalar(prec.tag, 0.0)
        self.stream = torch.cuda.current_stream().cuda_stream
        lib = _lib.load()
        t = prec.tag
        if kernel in ("symv", "hemv"):
            name = {"s": "ssymv", "d": "dsymv"}.get(t) or (f"{t}hemv" if kernel == "hemv" else f"{t}symv")
            self.fn = getattr(lib, f"kblas_{name}_async")
            self.args = lambda A: (uplo.encode(), n, self.one, A.data_ptr(), n, self.x.data_ptr(), 1, self.zero,
                                   self.y.data_ptr(), 1, self.stream)
        else:
            self.fn = getattr(lib, f"kblas_{t}gemv_async")
            trans = op_of(kernel).encode()
            self.args = lambda A: (trans, n, n, self.one, A.data_ptr(), n, self.x.data_ptr(), 1, self.zero,
                                   self.y.data_ptr(), 1, self.stream)

    def close(self):
        # drop the operands now (the argument closures refer back to self)
        self.As, self.x, self.y, self.args = [], None, None, None

    def call(self, i: int = 0):
        rc = self.fn(*self.args(self.As[i % len(self.As)]))
        _lib.check(rc, f"tuner {self.kernel}")

    def result(self):
        self.call(0)
        self.torch.cuda.synchronize()
        return self.y.clone()

    def time(self, reps: int, warmup: int) -> float:
        """Seconds per call, back to back over the rotating copies."""
        torch = self.torch
        for i in range(warmup):
            self.call(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(reps):
            self.call(i)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3 / reps


def _alg_bytes(kernel: str, prec: Precision, n: int) -> int:
    from .roofline import byte_count

    return byte_count(prec, "symv" if kernel in ("symv", "hemv") else "gemv", n)


def sweep(kernel: str, prec: Precision, sizes, configs, uplo: str = "l", reps: int = 20, warmup: int = 3,
          seed: int = 0, passes: int = 3) -> list[TunePoint]:
    """Time every config at every size on the current CUDA device (best of
    `passes` interleaved passes of `reps` back-to-back calls).  The
    library's tuning table is restored afterwards."""
    _check_kernel(kernel, prec)
    import torch

    op = op_of(kernel, uplo)
    saved = table()
    points = []
    try:
        for n in sorted(set(int(s) for s in sizes)):
            if n <= 0:
                raise ValueError(f"sizes must be positive, got {n}")
            b = _Bench(kernel, prec, n, uplo, seed)
            nbytes = _alg_bytes(kernel, prec, n)
            ref = None
            diffs, plans = [], []

            def install(cfg):
                restore(saved)
                if not cfg.is_auto:
                    set_entry(TableEntry(prec.tag, op, n, n, cfg.shape, cfg.form, cfg.waves))

            for cfg in configs:
                install(cfg)
                y = b.result()
                plans.append(_lib.last_plan())
                if ref is None:
                    ref = y
                diffs.append(float((y - ref).abs().max()) / (float(ref.abs().max()) or 1.0))
            # timing passes interleave the candidates so clock or thermal
            # drift does not favour the ones measured first; best pass wins
            best = [float("inf")] * len(configs)
            for _ in range(passes):
                for i, cfg in enumerate(configs):
                    install(cfg)
                    best[i] = min(best[i], b.time(reps, warmup))
            for i, cfg in enumerate(configs):
                points.append(TunePoint(kernel, prec, n, cfg, nbytes / best[i] / 1e9, best[i], diffs[i], plans[i],
                                        uplo))
            b.close()
            del b
            torch.cuda.empty_cache()
    finally:
        restore(saved)
    return points


def _rel_tol(prec: Precision, n: int) -> float:
    # different reduction orders of the same sums: a few ulps times sqrt(n)
    return 64 * prec.eps * math.sqrt(n)


def _pick(points: list[TunePoint], min_gain: float) -> TuneConfig:
    """Fastest correct config of one size; the first point (the built-in
    choice) keeps its place unless beaten by more than min_gain."""
    base = points[0]
    ok = [p for p in points if p.rel_diff <= _rel_tol(p.precision, p.size)]
    best = max(ok, key=lambda p: p.measured_gbs)
    if best is base or best.measured_gbs <= base.measured_gbs * (1 + min_gain):
        return base.config
    return best.config


def coarse_tune(kernel: str, prec: Precision, sizes, uplo: str = "l", reps: int = 20, warmup: int = 3,
                min_gain: float = 0.01) -> CoarseResult:
    """Stage one: the form left to the built-in rule, pick the shape that
    wins at the largest size (reference: coarse_tune, tuner.py:168-192)."""
    sizes = sorted(set(sizes))
    if not sizes:
        raise ValueError("coarse_tune needs at least one size")
    points = sweep(kernel, prec, [sizes[-1]], enumerate_configs(kernel, "coarse"), uplo, reps, warmup)
    w = _pick(points, min_gain)
    if op_of(kernel, uplo) in ("t", "c") and not w.is_auto:
        w = TuneConfig(w.shape)  # the fine stage scans the forms
    return CoarseResult(winner=w, points=points)


def fine_tune(kernel: str, prec: Precision, sizes, base: TuneConfig | None = None, uplo: str = "l",
              reps: int = 20, warmup: int = 3, min_gain: float = 0.01) -> FineResult:
    """Stage two: keep the coarse shape and pick the form per size (SYMV /
    HEMV: the shape per size).  The recommendation is the winner at the
    largest size (reference: fine_tune, tuner.py:195-235)."""
    sizes = sorted(set(sizes))
    if not sizes:
        raise ValueError("fine_tune needs at least one size")
    shape = None if base is None else base.shape
    configs = enumerate_configs(kernel, "fine", shape)
    points = sweep(kernel, prec, sizes, configs, uplo, reps, warmup)
    per_size = {}
    for n in sizes:
        per_size[n] = _pick([p for p in points if p.size == n], min_gain)
    return FineResult(kernel, prec, uplo, per_size, per_size[sizes[-1]], points)


def tune(kernel: str, prec_tag: str, sizes, uplo: str = "l", reps: int = 20, warmup: int = 3,
         min_gain: float = 0.01) -> tuple[CoarseResult, FineResult]:
    """Full two-stage pipeline; returns both stages' results (reference:
    tune, tuner.py:257-270)."""
    prec = precision(prec_tag)
    _check_kernel(kernel, prec)
    coarse = coarse_tune(kernel, prec, sizes, uplo, reps, warmup, min_gain)
    fine = fine_tune(kernel, prec, sizes, coarse.winner, uplo, reps, warmup, min_gain)
    return coarse, fine


SWEEP_CSV_HEADER = ["kernel", "precision", "uplo", "shape", "form", "waves", "size", "measured_gbs", "seconds",
                    "rel_diff", "plan"]


def write_sweep_csv(points, fh) -> None:
    """One row per measured point (reference: write_sweep_csv,
    tuner.py:238-254, with measured columns in place of predicted ones)."""
    w = csv.writer(fh)
    w.writerow(SWEEP_CSV_HEADER)
    for p in points:
        w.writerow([p.kernel, p.precision.tag, p.uplo, p.config.shape, p.config.form, p.config.waves, p.size,
                    f"{p.measured_gbs:.1f}", f"{p.seconds:.9f}", f"{p.rel_diff:.3e}", p.plan])
