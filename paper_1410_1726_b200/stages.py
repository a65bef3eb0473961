"""The reference's per-stage kernel entry points on the B200 kernels.

blockmv exposes the stages its gemv / symv_hemv are built from
(kernels.py:65-97 `KernelRequest`, 127-146 `run_scal`, 209-236
`run_gemv_n` / `run_gemv_t`, 287-313 `run_symv_offdiag`, 362-392
`run_diag_block`).  On B200 those stages are fused: one GEMV
launch sequence computes alpha*op(A)x + beta*y with beta in its epilogue,
and one streaming kernel reads every stored element of a triangle once for
both of its products, diagonal blocks included.  These functions keep the
stage decomposition for callers that drive the stages themselves, with the
reference's argument meaning, results and errors, each stage running on
the library's kernels through the C ABI:

  run_scal          the scal kernel (gemv with alpha = 0)
  run_gemv_n / _t   the GEMV kernels with beta = 1 (y + alpha*op(A)x)
  run_diag_block    the SYMV/HEMV kernels on each nb x nb diagonal block
                    (offset entry point), beta fused as in the reference
  run_symv_offdiag  for every block column, the GEMV-N and GEMV-T/C
                    kernels on its off-diagonal panel of the stored
                    triangle, accumulated in place (y + alpha*A_hat x
                    minus the diagonal blocks)

The report counters follow the reference formulas for flops
(kernels.py:204-206, 302-311, 355-357, 387-391) and the algorithmic bytes
of DESIGN.md §4 for traffic.  Nothing here runs on the CPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib, _ops
from .core import HermitianView, MatrixView, Precision
from .kernels import ExecutionReport, Op, _segs
from .partition import KernelConfig

_SYM_OPS = (Op.SYMV_LOWER, Op.SYMV_UPPER, Op.HEMV_LOWER, Op.HEMV_UPPER)


@dataclass
class KernelRequest:
    """One stage launch (kernels.py:65-97): op, operand, vectors, scalars
    and the reference's launch configuration (its block size sets the
    diagonal-block / panel width of the SYMV stages)."""

    op: Op
    a: MatrixView | HermitianView
    x: object
    y: object
    alpha: complex
    beta: complex
    config: KernelConfig

    def __post_init__(self):
        view = self.a.base if isinstance(self.a, HermitianView) else self.a
        m, n = view.rows, view.cols
        if self.op in (Op.GEMV_N, Op.GEMV_T):
            want_x, want_y = (n, m) if self.op is Op.GEMV_N else (m, n)
        else:
            if m != n:
                raise ValueError(f"symmetric ops need a square matrix, got {m}x{n}")
            if not isinstance(self.a, HermitianView):
                raise ValueError("symmetric/hermitian ops require a HermitianView")
            want_x = want_y = n
        if len(self.x) != want_x:
            raise ValueError(f"x has length {len(self.x)}, expected {want_x}")
        if len(self.y) != want_y:
            raise ValueError(f"y has length {len(self.y)}, expected {want_y}")

    @property
    def view(self) -> MatrixView:
        return self.a.base if isinstance(self.a, HermitianView) else self.a

    @property
    def precision(self) -> Precision:
        return self.view.precision


def _device_of(*objs):
    return _ops.device_for(*objs)


def _vec_bytes(rep: ExecutionReport, n: int, eb: int, read: bool = True, written: bool = False):
    if read:
        rep.bytes_read += n * eb
        rep.transactions += _segs(n * eb)
    if written:
        rep.bytes_written += n * eb
        rep.transactions += _segs(n * eb)


def run_scal(y, beta, prec: Precision) -> ExecutionReport:
    """y <- beta * y as a standalone kernel (kernels.py:127-146); beta == 0
    writes zeros without reading y, so NaN/Inf in y cannot propagate."""
    rep = ExecutionReport()
    n = len(y)
    eb = prec.element_bytes
    if n == 0:
        rep.y_out = _ops.result_like(y, torch.empty(0, dtype=prec.torch_dtype, device=_device_of(y)))
        return rep
    dev = _device_of(y)
    bz = complex(beta) == 0
    out = _ops.output_vector(y, n, prec, dev, bz, False)
    dummy = torch.empty(1, dtype=prec.torch_dtype, device=dev)
    # gemv with alpha = 0 is the library's scal kernel (A is not read)
    _ops.call_gemv(prec, "n", n, 1, 0.0, 0, max(1, n), dummy, beta, out, dev)
    rep.y_out = _ops.result_like(y, out)
    rep.flops += prec.flops_per_mul * n
    if not bz:
        _vec_bytes(rep, n, eb)
    _vec_bytes(rep, n, eb, read=False, written=True)
    rep.tb_count += -(-n // 256)
    rep.plan = _lib.last_plan()
    return rep


def _gemv_stage(req: KernelRequest, trans: str) -> ExecutionReport:
    view = req.view
    prec = view.precision
    m, n = view.rows, view.cols
    x_len, y_len = (n, m) if trans == "n" else (m, n)
    dev = _device_of(view, req.y, req.x)
    xd = _ops.vector_in(req.x, x_len, prec, "x", dev)
    out = _ops.output_vector(req.y, y_len, prec, dev, False, False)
    rep = ExecutionReport()
    if m and n and complex(req.alpha) != 0:
        ptr, lda, keep = _ops.matrix_in(view, dev)
        _ops.call_gemv(prec, trans, m, n, req.alpha, ptr, lda, xd, 1.0, out, dev)
        rep.plan = _lib.last_plan()
        del keep
    eb = prec.element_bytes
    rep.bytes_read += m * n * eb
    rep.matrix_transactions += _segs(m * n * eb)
    rep.transactions += rep.matrix_transactions
    _vec_bytes(rep, x_len, eb)
    _vec_bytes(rep, y_len, eb, read=True, written=True)
    # products m*n, dot-reduction adds, alpha scaling, merge adds (kernels.py:204-206)
    o, i = y_len, x_len
    rep.flops += prec.flops_per_mul * (o * i + o) + prec.flops_per_add * (o * i)
    rep.y_out = _ops.result_like(req.y, out)
    return rep


def run_gemv_n(req: KernelRequest) -> ExecutionReport:
    """Accumulation stage y + alpha*A x (kernels.py:209-221; beta is
    run_scal's)."""
    if req.op is not Op.GEMV_N:
        raise ValueError(f"expected GEMV_N request, got {req.op}")
    return _gemv_stage(req, "n")


def run_gemv_t(req: KernelRequest, conjugate: bool = False) -> ExecutionReport:
    """Accumulation stage y + alpha*A^T x (A^H with `conjugate`;
    kernels.py:224-236)."""
    if req.op is not Op.GEMV_T:
        raise ValueError(f"expected GEMV_T request, got {req.op}")
    return _gemv_stage(req, "c" if conjugate and req.precision.is_complex else "t")


def _sym_setup(req: KernelRequest):
    if req.op not in _SYM_OPS:
        raise ValueError(f"expected a symmetric/hermitian request, got {req.op}")
    hv = req.a
    view = hv.base
    prec = view.precision
    hermitian = req.op in (Op.HEMV_LOWER, Op.HEMV_UPPER)
    if hermitian and not prec.is_complex:
        raise ValueError("hermitian treatment requires a complex precision")
    d = hv.dim
    dev = _device_of(view, req.y, req.x)
    return hv, view, prec, hermitian, d, dev


def run_diag_block(req: KernelRequest) -> ExecutionReport:
    """Diagonal-block stage with beta fused (kernels.py:362-392): for each
    nb x nb diagonal block, alpha * D x + beta * y on its segment, D the
    stored triangle mirrored (conjugated, diagonal real for HEMV).  Runs
    the SYMV/HEMV kernels on each block through the offset entry point."""
    hv, view, prec, hermitian, d, dev = _sym_setup(req)
    nb = req.config.block_size
    xd = _ops.vector_in(req.x, d, prec, "x", dev)
    bz = complex(req.beta) == 0
    out = _ops.output_vector(req.y, d, prec, dev, bz, False)
    rep = ExecutionReport()
    ptr, lda, keep = _ops.matrix_in(view, dev, lower_tri=hv.uplo)
    eb = prec.element_bytes
    for r0 in range(0, d, nb):
        rb = min(d, r0 + nb) - r0
        _ops.call_symv(prec, hermitian, hv.uplo, rb, req.alpha, ptr, lda, xd[r0:r0 + rb], req.beta,
                       out[r0:r0 + rb], dev, offset=r0)
        rep.flops += prec.flops_per_mul * (rb * rb + rb) + prec.flops_per_add * (rb * rb)
        rep.bytes_read += rb * (rb + 1) // 2 * eb
        rep.tb_count += 1
    del keep
    rep.matrix_transactions += _segs(rep.bytes_read)
    rep.transactions += rep.matrix_transactions
    _vec_bytes(rep, d, eb)
    _vec_bytes(rep, d, eb, read=not bz, written=True)
    rep.flops += prec.flops_per_mul * d  # nominal beta scaling (kernels.py:387)
    rep.plan = _lib.last_plan()
    rep.y_out = _ops.result_like(req.y, out)
    return rep


def run_symv_offdiag(req: KernelRequest) -> ExecutionReport:
    """Off-diagonal stage y + alpha * (A_hat - D) x from one stored triangle
    (kernels.py:287-313): every stored block outside the diagonal blocks
    contributes once as stored (GEMV-N on its panel) and once transposed /
    conjugate-transposed (GEMV-T/C), accumulated in place on the device."""
    hv, view, prec, hermitian, d, dev = _sym_setup(req)
    nb = req.config.block_size
    xd = _ops.vector_in(req.x, d, prec, "x", dev)
    out = _ops.output_vector(req.y, d, prec, dev, False, False)
    rep = ExecutionReport()
    ptr, lda, keep = _ops.matrix_in(view, dev, lower_tri=hv.uplo)
    lower = hv.uplo == "l"
    tr = "c" if hermitian else "t"
    eb = prec.element_bytes
    if complex(req.alpha) != 0:
        for c0 in range(0, d, nb):
            c1 = min(d, c0 + nb)
            r0, r1 = (c1, d) if lower else (0, c0)
            rows = r1 - r0
            if rows <= 0:
                continue
            # stored panel A[r0:r1, c0:c1]: y[r] += alpha * P x[c]; y[c] += alpha * P^T|H x[r]
            _ops.call_gemv(prec, "n", rows, c1 - c0, req.alpha, ptr, lda, xd[c0:c1], 1.0, out[r0:r1], dev,
                           off_r=r0, off_c=c0)
            _ops.call_gemv(prec, tr, rows, c1 - c0, req.alpha, ptr, lda, xd[r0:r1], 1.0, out[c0:c1], dev,
                           off_r=r0, off_c=c0)
            rep.bytes_read += rows * (c1 - c0) * eb
            rep.tb_count += 1
        rep.plan = _lib.last_plan()
    del keep
    t = -(-d // nb)
    diag_elems = (t - 1) * nb * nb + (d - (t - 1) * nb) ** 2
    off = d * d - diag_elems
    rep.flops += prec.flops_per_mul * off + prec.flops_per_add * off
    rep.matrix_transactions += _segs(rep.bytes_read)
    rep.transactions += rep.matrix_transactions
    _vec_bytes(rep, d, eb)
    _vec_bytes(rep, d, eb, read=True, written=True)
    rep.y_out = _ops.result_like(req.y, out)
    return rep


__all__ = ["KernelRequest", "run_scal", "run_gemv_n", "run_gemv_t", "run_diag_block", "run_symv_offdiag"]
