"""Submatrix ("new interface") GEMV and SYMV/HEMV (offset.py:37-208).

The caller passes the parent matrix and the submatrix position, as in the
paper.  The reference reads an nb-aligned frame and
zero-masks it (offset.py:66-71,109-114).  On B200 the C ABI takes the
parent pointer plus (offset_r, offset_c), realigns the first row down to
its 32-byte load granule and masks only the lead rows in registers;
columns need no padding because a column's start depends on ld alone.
Numerically it equals the standard kernel on the extracted submatrix.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

from . import _lib, _ops, roofline
from .core import HermitianView, MatrixView
from .kernels import SEGMENT_BYTES, ExecutionReport, _DeferredReport, _is_one, _is_zero, _scal_report, fill_report
from .partition import DEFAULT_CONFIG, KernelConfig


@dataclass(frozen=True)
class OffsetRequest:
    """A submatrix operation described against the parent (offset.py:37-51)."""

    parent: MatrixView
    row_off: int
    col_off: int
    sub_m: int
    sub_n: int

    def __post_init__(self):
        if self.row_off < 0 or self.col_off < 0 or self.sub_m <= 0 or self.sub_n <= 0:
            raise ValueError("offsets must be >= 0 and submatrix dimensions positive")
        if self.row_off + self.sub_m > self.parent.rows or self.col_off + self.sub_n > self.parent.cols:
            raise ValueError("submatrix exceeds the parent matrix")


def effective_dims(m: int, n: int, sub_m: int, sub_n: int, nb: int) -> tuple[int, int]:
    """Eq. 9: requested dims padded to the next nb multiple, capped at the parent (offset.py:54-63)."""
    if sub_m > m or sub_n > n:
        raise ValueError("submatrix dimensions exceed the parent")
    if sub_m <= 0 or sub_n <= 0 or nb <= 0:
        raise ValueError("dimensions and nb must be positive")
    pad_m = min(m, -(-sub_m // nb) * nb)
    pad_n = min(n, -(-sub_n // nb) * nb)
    return pad_m, pad_n


def realigned_frame(row_off: int, sub_m: int, element_bytes: int, granule: int = 32) -> tuple[int, int, int]:
    """(aligned_start, frame_rows, lead) of the B200 row realignment: start at
    the load granule at or below row_off (assuming a granule-aligned parent
    column), lead < granule / element_bytes rows masked."""
    per = max(1, granule // element_bytes)
    start = row_off - row_off % per
    lead = row_off - start
    return start, lead + sub_m, lead


def _check_alignment(parent: MatrixView):
    # same warning as offset.py:74-80 (message kept for drop-in callers)
    if (parent.ld * parent.precision.element_bytes) % SEGMENT_BYTES != 0:
        warnings.warn(
            "parent leading dimension is not segment-aligned; offset kernel reads "
            "will still be counted against the unaligned addresses",
            stacklevel=3,
        )


def gemv_offset(trans: str, alpha, req: OffsetRequest, x, beta, y,
                config: KernelConfig = DEFAULT_CONFIG) -> ExecutionReport:
    """GEMV on req's submatrix through kblas_xgemv_offset (offset.py:83-143)."""
    trans = trans.lower()
    if trans not in ("n", "t", "c"):
        raise ValueError(f"trans must be 'n', 't' or 'c', got {trans!r}")
    parent = req.parent
    prec = parent.precision
    if trans == "c" and not prec.is_complex:
        trans = "t"
    _check_alignment(parent)
    x_len, y_len = (req.sub_n, req.sub_m) if trans == "n" else (req.sub_m, req.sub_n)
    dev = _ops.device_for(parent, y, x)
    if _ops.host_vectors(x, y, False) and not _is_zero(alpha):
        # numpy x and y: one kblas_mv_hostvec call with the offsets
        ptr, lda, keep = _ops.matrix_in(parent, dev)
        try:
            y_out, plan = _ops.call_hostvec(prec, "g", trans, False, req.sub_m, req.sub_n, alpha, ptr, lda, x,
                                            x_len, beta, y, y_len, dev, off_r=req.row_off, off_c=req.col_off)
        except ValueError as e:
            if "vector of length" not in str(e):
                raise
            raise ValueError(f"expected x of length {x_len} and y of length {y_len}") from None
        del keep

        def report():
            r = ExecutionReport()
            fill_report(r, prec, req.sub_m * req.sub_n, x_len, y_len, _is_zero(beta),
                        roofline.gemv_flops(prec, req.sub_m, req.sub_n, trans), plan)
            r.scal_invocations = 1
            return r

        return _DeferredReport(y_out, report)
    try:
        xd = _ops.vector_in(x, x_len, prec, "x", dev)
        bz = _is_zero(beta)
        if _is_zero(alpha) and _is_one(beta):
            return ExecutionReport(y_out=_ops.result_like(y, _ops.vector_in(y, y_len, prec, "y", dev).clone()))
        out = _ops.output_vector(y, y_len, prec, dev, bz, False)
    except ValueError:
        raise ValueError(f"expected x of length {x_len} and y of length {y_len}")
    if _is_zero(alpha):
        _ops.call_gemv(prec, trans, req.sub_m, req.sub_n, alpha, 0, max(1, req.sub_m), xd, beta, out, dev)
        rep = _scal_report(prec, y_len, bz)
        rep.scal_invocations = 1
        rep.y_out = _ops.result_like(y, out)
        return rep
    ptr, lda, keep = _ops.matrix_in(parent, dev)
    _ops.call_gemv(prec, trans, req.sub_m, req.sub_n, alpha, ptr, lda, xd, beta, out, dev,
                   off_r=req.row_off, off_c=req.col_off)
    rep = ExecutionReport()
    fill_report(rep, prec, req.sub_m * req.sub_n, x_len, y_len, bz,
                roofline.gemv_flops(prec, req.sub_m, req.sub_n, trans), _lib.last_plan())
    rep.scal_invocations = 1
    rep.y_out = _ops.result_like(y, out)
    del keep
    return rep


def symv_hemv_offset(uplo: str, alpha, parent: HermitianView, offset: int, sub_d: int, x, beta, y,
                     config: KernelConfig = DEFAULT_CONFIG, hermitian: bool | None = None) -> ExecutionReport:
    """SYMV/HEMV on the diagonal submatrix at (offset, offset) (offset.py:146-208)."""
    uplo = uplo.lower()
    if uplo != parent.uplo:
        raise ValueError(f"uplo {uplo!r} does not match the stored triangle {parent.uplo!r}")
    prec = parent.base.precision
    if hermitian is None:
        hermitian = prec.is_complex
    if hermitian and not prec.is_complex:
        raise ValueError("hermitian treatment requires a complex precision")
    if offset < 0 or sub_d <= 0 or offset + sub_d > parent.dim:
        raise ValueError("submatrix exceeds the parent matrix")
    _check_alignment(parent.base)
    dev = _ops.device_for(parent.base, y, x)
    if _ops.host_vectors(x, y, False) and not _is_zero(alpha):
        # numpy x and y: one kblas_mv_hostvec call at (offset, offset)
        ptr, lda, keep = _ops.matrix_in(parent.base, dev, lower_tri=uplo)
        try:
            y_out, plan = _ops.call_hostvec(prec, "s", uplo, hermitian, sub_d, sub_d, alpha, ptr, lda, x, sub_d,
                                            beta, y, sub_d, dev, off_r=offset, off_c=offset)
        except ValueError as e:
            if "vector of length" not in str(e):
                raise
            raise ValueError(f"expected x and y of length {sub_d}") from None
        del keep

        def report():
            r = ExecutionReport()
            fill_report(r, prec, sub_d * (sub_d + 1) // 2, sub_d, sub_d, _is_zero(beta),
                        roofline.symv_flops(prec, sub_d), plan)
            return r

        return _DeferredReport(y_out, report)
    try:
        xd = _ops.vector_in(x, sub_d, prec, "x", dev)
        bz = _is_zero(beta)
        if _is_zero(alpha) and _is_one(beta):
            return ExecutionReport(y_out=_ops.result_like(y, _ops.vector_in(y, sub_d, prec, "y", dev).clone()))
        out = _ops.output_vector(y, sub_d, prec, dev, bz, False)
    except ValueError:
        raise ValueError(f"expected x and y of length {sub_d}")
    if _is_zero(alpha):
        _ops.call_symv(prec, hermitian, uplo, sub_d, alpha, 0, max(1, sub_d), xd, beta, out, dev)
        rep = _scal_report(prec, sub_d, bz)
        rep.y_out = _ops.result_like(y, out)
        return rep
    ptr, lda, keep = _ops.matrix_in(parent.base, dev, lower_tri=uplo)
    _ops.call_symv(prec, hermitian, uplo, sub_d, alpha, ptr, lda, xd, beta, out, dev, offset=offset)
    rep = ExecutionReport()
    fill_report(rep, prec, sub_d * (sub_d + 1) // 2, sub_d, sub_d, bz, roofline.symv_flops(prec, sub_d),
                _lib.last_plan())
    rep.y_out = _ops.result_like(y, out)
    del keep
    return rep
