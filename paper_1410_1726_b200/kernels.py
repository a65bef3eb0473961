"""Standard-interface GEMV / SYMV / HEMV on B200.

Same names, argument meaning and error behaviour as blockmv.kernels
(kernels.py:402-500); the work happens in the sm_100a kernels behind the C
ABI (include/kblas_b200.h).  There is no CPU path: without the library or
a CUDA device these functions raise.

Semantics kept from the reference:
  * 'c' on a real precision is 't' (kernels.py:422-423); trans/uplo are
    case-insensitive; bad values raise ValueError with the same messages.
  * x, y are cast to the precision dtype and length-checked (395-399).
  * alpha == 0 and beta == 1 returns a copy of y, nothing launched (427-428).
  * beta == 0 writes y without reading it, so NaN/Inf in y never propagate.
  * Inputs are never mutated; y_out is a fresh vector (numpy in -> numpy
    out, torch in -> torch out), unless ``inplace=True`` on a CUDA tensor.
Deliberate difference: symv/hemv with alpha == 0
scale y without reading A (BLAS semantics); the reference still runs its
diagonal kernel (kernels.py:480-482), which only differs for non-finite A.

`ExecutionReport` keeps the reference's ten fields.  flops follows the
reference formulas exactly; byte and transaction fields are the
algorithmic traffic; tb_count is the CTAs actually
launched; atomic_adds is 0 (every cross-CTA sum is a fixed-order two-pass
reduction); scal_invocations is 1 for GEMV (the beta stage, fused into
the epilogue kernel) and 0 for SYMV/HEMV, as in the reference.
"""

from __future__ import annotations

import enum
import re
from dataclasses import dataclass, fields

from . import _lib, _ops, roofline
from .core import HermitianView, MatrixView, Precision
from .partition import DEFAULT_CONFIG, KernelConfig

SEGMENT_BYTES = 128


class Op(enum.Enum):
    GEMV_N = "gemv-n"
    GEMV_T = "gemv-t"
    SYMV_LOWER = "symv-lower"
    SYMV_UPPER = "symv-upper"
    HEMV_LOWER = "hemv-lower"
    HEMV_UPPER = "hemv-upper"


@dataclass
class ExecutionReport:
    """Result vector plus counters for one call (kernels.py:37-62)."""

    y_out: object = None
    bytes_read: int = 0
    bytes_written: int = 0
    transactions: int = 0
    matrix_transactions: int = 0
    flops: int = 0
    atomic_adds: int = 0
    tb_count: int = 0
    reduction_events: int = 0
    scal_invocations: int = 0
    plan: str = ""

    def absorb(self, other: "ExecutionReport"):
        self.bytes_read += other.bytes_read
        self.bytes_written += other.bytes_written
        self.transactions += other.transactions
        self.matrix_transactions += other.matrix_transactions
        self.flops += other.flops
        self.atomic_adds += other.atomic_adds
        self.tb_count += other.tb_count
        self.reduction_events += other.reduction_events
        self.scal_invocations += other.scal_invocations


class _DeferredReport(ExecutionReport):
    """ExecutionReport of a numpy-vector call whose counters are computed on
    first access (the call itself only records the launch plan), so the
    bookkeeping costs nothing on the call path when nobody reads it.  It
    compares equal to an ExecutionReport with the same fields, and pickles
    and copies (dataclasses.replace included) as an ExecutionReport."""

    def __init__(self, y_out=None, fill=None, **fields_):
        if fill is None:  # dataclasses.replace / plain construction
            super().__init__(y_out=y_out, **fields_)
            return
        self.__dict__["_fill"] = fill
        self.y_out = y_out

    def _materialize(self):
        fill = self.__dict__.pop("_fill", None)
        if fill is not None:
            rep = fill()
            for name in _COUNTER_FIELDS:
                self.__dict__.setdefault(name, rep.__dict__[name])

    def _as_tuple(self):
        return tuple(getattr(self, f.name) for f in fields(ExecutionReport))

    def __eq__(self, other):
        if not isinstance(other, ExecutionReport):
            return NotImplemented
        return self._as_tuple() == tuple(getattr(other, f.name) for f in fields(ExecutionReport))

    __hash__ = None

    def __reduce__(self):
        self._materialize()
        rep = ExecutionReport(**{f.name: getattr(self, f.name) for f in fields(ExecutionReport)})
        extra = {k: v for k, v in self.__dict__.items() if k not in rep.__dict__ and k != "_fill"}
        return (ExecutionReport, (), {**rep.__dict__, **extra})


def _deferred_field(name):
    def get(self):
        d = self.__dict__
        if name not in d:
            self._materialize()
        return d[name]

    def put(self, value):
        self._materialize()
        self.__dict__[name] = value

    return property(get, put)


_COUNTER_FIELDS = [f.name for f in fields(ExecutionReport) if f.name != "y_out"]
for _name in _COUNTER_FIELDS:
    setattr(_DeferredReport, _name, _deferred_field(_name))


def _segs(nbytes: int) -> int:
    return -(-nbytes // SEGMENT_BYTES)


def _is_zero(v) -> bool:
    return complex(v) == 0


def _is_one(v) -> bool:
    return complex(v) == 1


_PLAN_CACHE: dict = {}


def plan_counters(plan: str) -> tuple[int, int]:
    """(CTAs of the main kernel, partial slots) parsed from kblas_last_plan()
    (memoised: a shape's plan string repeats from call to call)."""
    hit = _PLAN_CACHE.get(plan)
    if hit is not None:
        return hit
    p = re.search(r"\bP=(\d+)", plan)
    s = re.search(r"\bslots=(\d+)", plan)
    res = (int(p.group(1)) if p else 0, int(s.group(1)) if s else 0)
    if len(_PLAN_CACHE) < 4096:
        _PLAN_CACHE[plan] = res
    return res


def fill_report(rep: ExecutionReport, prec: Precision, mat_elems: int, x_len: int, y_len: int,
                beta_zero: bool, flops: int, plan: str):
    eb = prec.element_bytes
    rep.matrix_transactions = _segs(mat_elems * eb)
    rep.bytes_read = (mat_elems + x_len + (0 if beta_zero else y_len)) * eb
    rep.bytes_written = y_len * eb
    rep.transactions = rep.matrix_transactions + _segs(x_len * eb) + _segs(y_len * eb) * (1 if beta_zero else 2)
    rep.flops = flops
    rep.plan = plan
    ctas, slots = plan_counters(plan)
    # SYMV/HEMV add one epilogue CTA per 32 rows; GEMV's epilogue is fused
    rep.tb_count = ctas + (-(-y_len // 32) if plan.startswith("symv") else 0)
    rep.reduction_events = slots


def _scal_report(prec: Precision, y_len: int, beta_zero: bool) -> ExecutionReport:
    rep = ExecutionReport()
    fill_report(rep, prec, 0, 0, y_len, beta_zero, prec.flops_per_mul * y_len, _lib.last_plan())
    rep.tb_count = -(-y_len // 256)
    return rep


def gemv(trans: str, alpha, a: MatrixView, x, beta, y, config: KernelConfig = DEFAULT_CONFIG,
         inplace: bool = False, _keep: list | None = None) -> ExecutionReport:
    """y = alpha * op(A) x + beta * y, op in {n, t, c} (kernels.py:402-440)."""
    trans = trans.lower()
    if trans not in ("n", "t", "c"):
        raise ValueError(f"trans must be 'n', 't' or 'c', got {trans!r}")
    if not isinstance(a, MatrixView):
        raise ValueError("gemv requires a MatrixView")
    prec = a.precision
    if trans == "c" and not prec.is_complex:
        trans = "t"
    x_len, y_len = (a.cols, a.rows) if trans == "n" else (a.rows, a.cols)
    dev = _ops.device_for(a, y, x)
    if _ops.host_vectors(x, y, inplace) and not _is_zero(alpha):
        return _gemv_hostvec(trans, alpha, a, x, beta, y, prec, x_len, y_len, dev, _keep)
    xd = _ops.vector_in(x, x_len, prec, "x", dev)
    if _is_zero(alpha) and _is_one(beta):
        yd = _ops.vector_in(y, y_len, prec, "y", dev)
        out = yd if inplace else yd.clone()
        return ExecutionReport(y_out=_ops.result_like(y, out))
    bz = _is_zero(beta)
    out = _ops.output_vector(y, y_len, prec, dev, bz, inplace)
    if _is_zero(alpha):
        _ops.call_gemv(prec, trans, a.rows, a.cols, alpha, 0, max(1, a.rows), xd, beta, out, dev)
        rep = _scal_report(prec, y_len, bz)
        rep.scal_invocations = 1
        rep.y_out = _ops.result_like(y, out)
        return rep
    ptr, lda, keep = _ops.matrix_in(a, dev)
    _ops.call_gemv(prec, trans, a.rows, a.cols, alpha, ptr, lda, xd, beta, out, dev)
    rep = ExecutionReport()
    fill_report(rep, prec, a.rows * a.cols, x_len, y_len, bz,
                roofline.gemv_flops(prec, a.rows, a.cols, trans), _lib.last_plan())
    rep.scal_invocations = 1
    rep.y_out = _ops.result_like(y, out)
    del keep
    return rep


def _gemv_hostvec(trans, alpha, a: MatrixView, x, beta, y, prec, x_len, y_len, dev, keep_list=None) -> ExecutionReport:
    """numpy x and y: one kblas_mv_hostvec call (copies, kernels, result);
    keep_list not None: no wait (a queue submission, see gemv_async)."""
    ptr, lda, keep = _ops.matrix_in(a, dev)
    y_out, plan = _ops.call_hostvec(prec, "g", trans, False, a.rows, a.cols, alpha, ptr, lda, x, x_len, beta, y,
                                    y_len, dev, keep=keep_list)

    def report():
        rep = ExecutionReport()
        fill_report(rep, prec, a.rows * a.cols, x_len, y_len, _is_zero(beta),
                    roofline.gemv_flops(prec, a.rows, a.cols, trans), plan)
        rep.scal_invocations = 1
        return rep

    rep = _DeferredReport(y_out, report)
    if keep_list is not None:
        keep_list.append(keep)
    del keep
    return rep


def symv_hemv(uplo: str, alpha, a: HermitianView, x, beta, y, config: KernelConfig = DEFAULT_CONFIG,
              hermitian: bool | None = None, inplace: bool = False, _keep: list | None = None) -> ExecutionReport:
    """y = alpha * A x + beta * y from one stored triangle (kernels.py:443-486)."""
    if not isinstance(a, HermitianView):
        raise ValueError("symv/hemv requires a HermitianView")
    uplo = uplo.lower()
    if uplo not in ("l", "u"):
        raise ValueError(f"uplo must be 'l' or 'u', got {uplo!r}")
    if uplo != a.uplo:
        raise ValueError(f"uplo {uplo!r} does not match the stored triangle {a.uplo!r}")
    prec = a.base.precision
    if hermitian is None:
        hermitian = prec.is_complex
    if hermitian and not prec.is_complex:
        raise ValueError("hermitian treatment requires a complex precision")
    d = a.dim
    dev = _ops.device_for(a.base, y, x)
    if _ops.host_vectors(x, y, inplace) and not _is_zero(alpha):
        # numpy x and y: one kblas_mv_hostvec call (copies, kernels, result)
        ptr, lda, keep = _ops.matrix_in(a.base, dev, lower_tri=uplo)
        y_out, plan = _ops.call_hostvec(prec, "s", uplo, hermitian, d, d, alpha, ptr, lda, x, d, beta, y, d, dev,
                                        keep=_keep)

        def report():
            rep = ExecutionReport()
            fill_report(rep, prec, d * (d + 1) // 2, d, d, _is_zero(beta), roofline.symv_flops(prec, d), plan)
            return rep

        rep = _DeferredReport(y_out, report)
        if _keep is not None:
            _keep.append(keep)
        del keep
        return rep
    xd = _ops.vector_in(x, d, prec, "x", dev)
    if _is_zero(alpha) and _is_one(beta):
        yd = _ops.vector_in(y, d, prec, "y", dev)
        out = yd if inplace else yd.clone()
        return ExecutionReport(y_out=_ops.result_like(y, out))
    bz = _is_zero(beta)
    out = _ops.output_vector(y, d, prec, dev, bz, inplace)
    if _is_zero(alpha):
        _ops.call_symv(prec, hermitian, uplo, d, alpha, 0, max(1, d), xd, beta, out, dev)
        rep = _scal_report(prec, d, bz)
        rep.y_out = _ops.result_like(y, out)
        return rep
    ptr, lda, keep = _ops.matrix_in(a.base, dev, lower_tri=uplo)
    _ops.call_symv(prec, hermitian, uplo, d, alpha, ptr, lda, xd, beta, out, dev)
    rep = ExecutionReport()
    fill_report(rep, prec, d * (d + 1) // 2, d, d, bz, roofline.symv_flops(prec, d), _lib.last_plan())
    rep.y_out = _ops.result_like(y, out)
    del keep
    return rep


def symv(uplo, alpha, a, x, beta, y, config: KernelConfig = DEFAULT_CONFIG, **kw) -> ExecutionReport:
    """Real symmetric MV (kernels.py:489-493)."""
    if a.base.precision.is_complex:
        raise ValueError("symv supports real precisions; use hemv for complex matrices")
    return symv_hemv(uplo, alpha, a, x, beta, y, config, hermitian=False, **kw)


def hemv(uplo, alpha, a, x, beta, y, config: KernelConfig = DEFAULT_CONFIG, **kw) -> ExecutionReport:
    """Complex Hermitian MV (kernels.py:496-500)."""
    if not a.base.precision.is_complex:
        raise ValueError("hemv supports complex precisions; use symv for real matrices")
    return symv_hemv(uplo, alpha, a, x, beta, y, config, hermitian=True, **kw)


# ---------------------------------------------------------------------------
# Queued single-GPU calls (the reference's CommandQueue contract,
# multidevice.py:287-332, applied to gemv / symv_hemv): the call is enqueued
# on the queue's CUDA stream and returns a handle; `queue.synchronize()`
# waits, and `handle.result()` is the ExecutionReport.  With numpy x and y
# the per-call host wait disappears, so back-to-back calls pipeline (the
# copies, kernels and result writes of call i+1 are queued behind call i
# instead of each waiting on the host).  x must not be modified and the
# result not read before the queue has synchronised.
# ---------------------------------------------------------------------------
def gemv_async(trans, alpha, a, x, beta, y, config: KernelConfig = DEFAULT_CONFIG, queue=None):
    """gemv on `queue` (a multidevice.CommandQueue); returns its handle."""
    return _submit(queue, gemv, trans, alpha, a, x, beta, y, config)


def symv_hemv_async(uplo, alpha, a, x, beta, y, config: KernelConfig = DEFAULT_CONFIG, queue=None,
                    hermitian=None):
    """symv_hemv on `queue` (a multidevice.CommandQueue); returns its handle."""
    return _submit(queue, symv_hemv, uplo, alpha, a, x, beta, y, config, hermitian)


def _submit(queue, fn, *args):
    if queue is None:
        raise ValueError("an async call needs a CommandQueue")
    keep: list = []

    def run():
        rep = fn(*args, _keep=keep)
        rep._keepalive = keep  # operands the queued work still reads
        return rep

    return queue.submit(run)
