"""B200-native KBLAS dense matrix-vector library.

Drop-in for the hot path of the reference package `blockmv`
(/root/reference/pkg/src/blockmv/__init__.py:28-53): gemv (N/T/C),
symv / hemv / symv_hemv (upper/lower), gemv_offset / symv_hemv_offset and
the mgpu API (distribute, gather, gemv_mgpu, symv_hemv_mgpu, *_async,
CommandQueue), in s/d/c/z.  Compute runs in hand-written sm_100a CUDA
kernels behind a C ABI (include/kblas_b200.h, libkblas_b200.so); there is
no CPU fallback.
"""

from .core import (
    PRECISIONS,
    WARP_SIZE,
    HermitianView,
    MatrixView,
    Precision,
    alloc_matrix,
    make_padded_view,
    precision,
    precision_of,
    view_of,
)
from .kernels import SEGMENT_BYTES, ExecutionReport, Op, gemv, gemv_async, hemv, symv, symv_hemv, symv_hemv_async
from .multidevice import (
    CommandQueue,
    DistributedMatrix,
    distribute,
    gather,
    gemv_mgpu,
    gemv_mgpu_async,
    local_col_count,
    owned_block_cols,
    partial_mv,
    required_local_elements,
    symv_hemv_mgpu,
    symv_hemv_mgpu_async,
)
from .offset import OffsetRequest, effective_dims, gemv_offset, symv_hemv_offset
from .partition import KernelConfig, tb_share
from .roofline import byte_count, flop_count
from .stages import KernelRequest, run_diag_block, run_gemv_n, run_gemv_t, run_scal, run_symv_offdiag

__version__ = "0.1.0"

__all__ = [
    "PRECISIONS",
    "SEGMENT_BYTES",
    "WARP_SIZE",
    "CommandQueue",
    "DistributedMatrix",
    "ExecutionReport",
    "HermitianView",
    "KernelConfig",
    "KernelRequest",
    "MatrixView",
    "OffsetRequest",
    "Op",
    "Precision",
    "alloc_matrix",
    "byte_count",
    "distribute",
    "effective_dims",
    "flop_count",
    "gather",
    "gemv",
    "gemv_async",
    "gemv_mgpu",
    "gemv_mgpu_async",
    "gemv_offset",
    "hemv",
    "local_col_count",
    "make_padded_view",
    "owned_block_cols",
    "partial_mv",
    "precision",
    "precision_of",
    "required_local_elements",
    "run_diag_block",
    "run_gemv_n",
    "run_gemv_t",
    "run_scal",
    "run_symv_offdiag",
    "symv",
    "symv_hemv",
    "symv_hemv_async",
    "symv_hemv_mgpu",
    "symv_hemv_mgpu_async",
    "symv_hemv_offset",
    "tb_share",
    "view_of",
]
