"""Precision table and column-major matrix descriptors.

Mirrors the reference's argument types (blockmv/core.py:27-188) so call
sites read the same: a `MatrixView` is an (offset, leading-dimension)
window into one flat buffer and never copies (core.py:66-132); a
`HermitianView` marks which triangle is stored (core.py:155-188).

Difference from the reference: `data` is normally a 1-D CUDA
`torch.Tensor` (HBM-resident operand).  A 1-D numpy array is also
accepted; the operation entry points then copy the referenced columns to
the GPU for the call (the host-buffer path timed as `e2e` by bench.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

WARP_SIZE = 32

_NP = {
    "s": np.dtype(np.float32),
    "d": np.dtype(np.float64),
    "c": np.dtype(np.complex64),
    "z": np.dtype(np.complex128),
}
_TORCH = {"s": torch.float32, "d": torch.float64, "c": torch.complex64, "z": torch.complex128}


@dataclass(frozen=True)
class Precision:
    """One of the four BLAS precisions (core.py:27-47)."""

    tag: str
    element_bytes: int
    flops_per_mul: int
    flops_per_add: int

    @property
    def is_complex(self) -> bool:
        return self.tag in ("c", "z")

    @property
    def dtype(self) -> np.dtype:
        return _NP[self.tag]

    @property
    def torch_dtype(self) -> torch.dtype:
        return _TORCH[self.tag]

    @property
    def eps(self) -> float:
        # epsilon of the real component type (core.py:44-47)
        return float(np.finfo(np.float32 if self.tag in ("s", "c") else np.float64).eps)


PRECISIONS = {
    "s": Precision("s", 4, 1, 1),
    "d": Precision("d", 8, 1, 1),
    "c": Precision("c", 8, 6, 2),
    "z": Precision("z", 16, 6, 2),
}


def precision(tag: str) -> Precision:
    """Look up a precision by tag, case-insensitive (core.py:58-63)."""
    try:
        return PRECISIONS[tag.lower()]
    except (KeyError, AttributeError):
        raise ValueError(f"unknown precision tag {tag!r}; expected one of s, d, c, z")


def precision_of(dtype) -> Precision:
    for tag in "sdcz":
        if dtype == _NP[tag] or dtype == _TORCH[tag]:
            return PRECISIONS[tag]
    raise ValueError(f"unsupported dtype {dtype}")


def _is_torch(a) -> bool:
    return isinstance(a, torch.Tensor)


@dataclass
class MatrixView:
    """A column-major rows x cols window of a flat parent buffer.

    Element (i, j) is ``data[(col_offset + j) * ld + row_offset + i]``
    (core.py:100-101).  Validation follows core.py:84-98.
    """

    data: object  # torch.Tensor (CUDA or CPU) | np.ndarray | None
    rows: int
    cols: int
    ld: int
    precision: Precision
    row_offset: int = 0
    col_offset: int = 0

    def __post_init__(self):
        if self.rows <= 0 or self.cols <= 0:
            raise ValueError(f"matrix dimensions must be positive, got {self.rows}x{self.cols}")
        if self.ld < self.rows + self.row_offset:
            raise ValueError(
                f"leading dimension {self.ld} too small for {self.rows} rows at offset {self.row_offset}"
            )
        if self.data is not None:
            needed = (self.col_offset + self.cols) * self.ld
            size = self.data.numel() if _is_torch(self.data) else self.data.size
            if self.data.ndim != 1 or size < needed:
                raise ValueError("parent buffer too small for the addressable region")
            want = self.precision.torch_dtype if _is_torch(self.data) else self.precision.dtype
            if self.data.dtype != want:
                raise ValueError(
                    f"buffer dtype {self.data.dtype} does not match precision {self.precision.tag}"
                )

    @property
    def on_device(self) -> bool:
        return _is_torch(self.data) and self.data.is_cuda

    def linear_index(self, i: int, j: int) -> int:
        return (self.col_offset + j) * self.ld + self.row_offset + i

    def decode_linear(self, index: int) -> tuple[int, int]:
        j, rem = divmod(index, self.ld)
        return rem - self.row_offset, j - self.col_offset

    def array(self):
        """Writable 2-D (rows x cols) view of the window, no copy."""
        if self.data is None:
            raise ValueError("geometry-only view has no element buffer")
        start = self.linear_index(0, 0)
        if _is_torch(self.data):
            return torch.as_strided(self.data, (self.rows, self.cols), (1, self.ld), start)
        itemsize = self.data.itemsize
        return np.lib.stride_tricks.as_strided(
            self.data[start:], shape=(self.rows, self.cols), strides=(itemsize, self.ld * itemsize)
        )

    def numpy(self) -> np.ndarray:
        """Host copy of the window (rows x cols)."""
        a = self.array()
        return a.detach().cpu().numpy().copy() if _is_torch(a) else np.array(a, copy=True)

    def submatrix(self, row_off: int, col_off: int, m: int, n: int) -> "MatrixView":
        if row_off < 0 or col_off < 0 or row_off + m > self.rows or col_off + n > self.cols:
            raise ValueError("submatrix exceeds parent window")
        return MatrixView(
            data=self.data,
            rows=m,
            cols=n,
            ld=self.ld,
            precision=self.precision,
            row_offset=self.row_offset + row_off,
            col_offset=self.col_offset + col_off,
        )


def _default_device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1410_1726_b200 needs a CUDA device (sm_100a); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def alloc_matrix(m: int, n: int, prec: Precision, ld: int | None = None, device=None) -> MatrixView:
    """Fresh zero-initialised column-major allocation (core.py:135-142),
    in HBM unless ``device="cpu"`` / ``device="numpy"``."""
    if m <= 0 or n <= 0:
        raise ValueError(f"matrix dimensions must be positive, got {m}x{n}")
    if ld is None:
        ld = m
    if device == "numpy":
        buf = np.zeros(ld * n, dtype=prec.dtype)
    else:
        dev = _default_device() if device is None else torch.device(device)
        buf = torch.zeros(ld * n, dtype=prec.torch_dtype, device=dev)
    return MatrixView(data=buf, rows=m, cols=n, ld=ld, precision=prec)


def make_padded_view(m: int, n: int, prec: Precision, pad_to: int, device=None) -> MatrixView:
    """Allocation whose ld is the smallest multiple of pad_to >= m (core.py:145-152)."""
    if pad_to <= 0:
        raise ValueError(f"pad_to must be positive, got {pad_to}")
    if m <= 0 or n <= 0:
        raise ValueError(f"matrix dimensions must be positive, got {m}x{n}")
    ld = -(-m // pad_to) * pad_to
    return alloc_matrix(m, n, prec, ld=ld, device=device)


def view_of(array, prec: Precision | None = None, ld: int | None = None) -> MatrixView:
    """Wrap a 2-D column-major (Fortran-ordered) array or a torch matrix as a view.

    torch tensors must have unit row stride (i.e. be a transposed
    row-major tensor, ``t.T`` of a contiguous tensor, or come from
    `MatrixView.array`)."""
    if _is_torch(array):
        if array.dim() != 2 or array.stride(0) != 1:
            raise ValueError("need a 2-D tensor with unit row stride (column-major)")
        prec = prec or precision_of(array.dtype)
        m, n = array.shape
        ld = ld or max(array.stride(1), m)
        # the reference's view covers n whole columns of ld elements
        # (core.py:92-94); a padded column-major tensor has them whenever its
        # storage extends past the last column's padding
        avail = array.untyped_storage().nbytes() // array.element_size() - array.storage_offset()
        length = n * ld if avail >= n * ld else (n - 1) * ld + m
        flat = torch.as_strided(array, (length,), (1,), array.storage_offset())
        return MatrixView(data=flat, rows=m, cols=n, ld=ld, precision=prec)
    a = np.asfortranarray(array)
    prec = prec or precision_of(a.dtype)
    m, n = a.shape
    return MatrixView(data=a.reshape(-1, order="F"), rows=m, cols=n, ld=m, precision=prec)


@dataclass
class HermitianView:
    """Square matrix with only one triangle meaningfully stored (core.py:155-188).

    The kernels never let an element of the unreferenced triangle into a
    sum: off-diagonal tiles of the wrong triangle are never loaded and the
    diagonal tiles mask it in registers.  ``guard`` is kept for API
    compatibility; ``violations`` therefore stays empty.  The executable
    check is to poison the other triangle with NaN and test the result is
    finite (tests/test_gpu_symv.py).
    """

    base: MatrixView
    uplo: str
    guard: bool = False
    violations: list = field(default_factory=list)

    def __post_init__(self):
        if self.base.rows != self.base.cols:
            raise ValueError("hermitian view requires a square window")
        self.uplo = self.uplo.lower()
        if self.uplo not in ("l", "u"):
            raise ValueError(f"uplo must be 'l' or 'u', got {self.uplo!r}")

    @property
    def dim(self) -> int:
        return self.base.rows

    def record_read(self, r0: int, r1: int, c0: int, c1: int, diag_block: bool = False):
        """Same contract as core.py:170-179 (used by host-side planners)."""
        if not self.guard or diag_block:
            return
        bad = (c1 - 1 > r0) if self.uplo == "l" else (r1 - 1 > c0)
        if bad:
            self.violations.append((r0, r1, c0, c1))
