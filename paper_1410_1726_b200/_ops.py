"""Operand marshalling between the Python API and the C ABI.

Shared by kernels.py, offset.py and multidevice.py: moves host operands to
HBM when needed, builds fresh output vectors (the reference never mutates
its inputs, SURVEY.md §8b "Ownership"), and calls the `_async` entry
points on the current torch stream.
"""

from __future__ import annotations

import sys
import threading

import numpy as np
import torch

from . import _lib
from .core import MatrixView, Precision, _is_torch

SYMV_FN = {("s", False): "ssymv", ("d", False): "dsymv", ("c", True): "chemv", ("z", True): "zhemv",
           ("c", False): "csymv", ("z", False): "zsymv"}


_CUDA_OK = False


def require_cuda():
    global _CUDA_OK
    if _CUDA_OK:
        return
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1410_1726_b200 needs a CUDA device (sm_100a); none is visible")
    _CUDA_OK = True


def device_for(*objs) -> torch.device:
    require_cuda()
    for o in objs:
        d = o.data if isinstance(o, MatrixView) else o
        if _is_torch(d) and d.is_cuda:
            return d.device
    return torch.device("cuda", torch._C._cuda_getDevice())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle(device) -> int:
    """cudaStream_t of torch's current stream on `device` (the raw accessor
    skips the Stream object construction, a few microseconds per call)."""
    idx = device.index if isinstance(device, torch.device) else device
    if _raw_stream is not None and idx is not None:
        return _raw_stream(idx)
    return torch.cuda.current_stream(device).cuda_stream


class _on_device:
    """`torch.cuda.device(d)` only when d is not already current (saves the
    context switch on the common path)."""

    __slots__ = ("dev", "prev")

    def __init__(self, dev):
        self.dev = dev.index if isinstance(dev, torch.device) else dev
        self.prev = None

    def __enter__(self):
        cur = torch._C._cuda_getDevice()
        if self.dev is not None and cur != self.dev:
            self.prev = cur
            torch.cuda.set_device(self.dev)

    def __exit__(self, *exc):
        if self.prev is not None:
            torch.cuda.set_device(self.prev)


def length_of(v) -> int:
    if _is_torch(v):
        return v.numel() if v.dim() == 1 else -1
    a = np.asarray(v)
    return a.size if a.ndim == 1 else -1


def output_vector(y_in, length: int, prec: Precision, device, beta_zero: bool, inplace: bool) -> torch.Tensor:
    """The buffer the kernels update: y itself (inplace), a fresh empty vector
    when beta == 0 (y is never read, so it is not even uploaded), else a
    private device copy of y."""
    if inplace:
        if not (_is_torch(y_in) and y_in.is_cuda and y_in.dim() == 1 and y_in.numel() == length
                and y_in.dtype == prec.torch_dtype and y_in.is_contiguous()):
            raise ValueError("inplace=True needs y to be a contiguous CUDA tensor of the operand dtype")
        return y_in
    if beta_zero:
        if length_of(y_in) != length:
            raise ValueError(f"y must be a vector of length {length}")
        return torch.empty(length, dtype=prec.torch_dtype, device=device)
    yd = vector_in(y_in, length, prec, "y", device)
    if _is_torch(y_in) and yd.data_ptr() == y_in.data_ptr():
        return yd.clone()
    return yd


def vector_in(v, length: int, prec: Precision, name: str, device) -> torch.Tensor:
    """1-D operand of the precision's dtype on `device` (kernels.py:395-399)."""
    if _is_torch(v):
        if v.dim() != 1 or v.numel() != length:
            raise ValueError(f"{name} must be a vector of length {length}")
        return v.to(device=device, dtype=prec.torch_dtype).contiguous()
    arr = np.asarray(v, dtype=prec.dtype)
    if arr.ndim != 1 or arr.size != length:
        raise ValueError(f"{name} must be a vector of length {length}")
    # non_blocking is safe for pageable memory too: the driver stages it
    # before returning, so the caller may reuse the array immediately
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device, non_blocking=True)


def result_like(y_in, y_out: torch.Tensor):
    """numpy in -> numpy out (one D2H read into a fresh page-locked buffer
    from torch's caching host allocator, so the copy is a direct DMA);
    torch in -> torch out (stays in HBM)."""
    if _is_torch(y_in):
        return y_out
    h = torch.empty(y_out.shape, dtype=y_out.dtype, pin_memory=True)
    h.copy_(y_out, non_blocking=True)
    torch.cuda.current_stream(y_out.device).synchronize()
    return h.numpy()


def matrix_in(view: MatrixView, device, lower_tri: str | None = None):
    """(device pointer of element (0, 0) of the view, lda, keepalive).

    A CUDA view is used in place.  Host data is copied column-wise: the
    view's columns (all ld rows, so the stride is kept) and, for a stored
    triangle, only the rows at or below ('l') / above ('u') each 256-column
    block's first column."""
    esize = view.precision.element_bytes
    if view.on_device:
        return view.data.data_ptr() + view.linear_index(0, 0) * esize, view.ld, view.data
    data = view.data
    host = data.numpy() if _is_torch(data) else data
    ld, c0, nc = view.ld, view.col_offset, view.cols
    src = np.ascontiguousarray(host[c0 * ld: (c0 + nc) * ld])
    dev = torch.empty(nc * ld, dtype=view.precision.torch_dtype, device=device)
    lib = _lib.load()
    st = stream_handle(device)
    hptr, dptr = src.ctypes.data, dev.data_ptr()
    r0 = view.row_offset
    with _on_device(device):
        if lower_tri is None:
            blocks = [(0, nc, 0, ld)]
        else:
            # only the stored triangle, 256-column blocks (SYMV/HEMV)
            blocks = []
            for b0 in range(0, nc, 256):
                b1 = min(nc, b0 + 256)
                lo, hi = (r0 + b0, r0 + view.rows) if lower_tri == "l" else (r0, r0 + b1)
                blocks.append((b0, b1, lo, hi))
        for b0, b1, lo, hi in blocks:
            off = (b0 * ld + lo) * esize
            _lib.check(lib.kblas_setmatrix_async(hi - lo, b1 - b0, esize, hptr + off, ld, dptr + off, ld, st),
                       "kblas_setmatrix_async")
        if not np.shares_memory(src, host):
            # a private staging copy must outlive the async copies
            torch.cuda.current_stream(device).synchronize()
    return dev.data_ptr() + view.row_offset * esize, ld, dev


INT_MAX = 2**31 - 1


def c_int_dims(what: str, **dims) -> None:
    """The C ABI takes BLAS-style 32-bit int dimensions, leading dimensions
    and offsets (include/kblas_b200.h); a larger value would wrap in the
    call, so it is rejected here (the reference's Python kernels have no
    such limit, so this is the one argument error the drop-in adds)."""
    for k, v in dims.items():
        if v > INT_MAX:
            raise ValueError(f"{what}: {k} = {v} exceeds the C ABI's 32-bit int range ({INT_MAX})")


_FN_CACHE: dict = {}


def _fn(name: str):
    f = _FN_CACHE.get(name)
    if f is None:
        f = _FN_CACHE[name] = getattr(_lib.load(), name)
    return f


def call_gemv(prec: Precision, trans: str, m: int, n: int, alpha, a_ptr: int, lda: int,
              x: torch.Tensor, beta, y: torch.Tensor, device, off_r: int = 0, off_c: int = 0):
    f = _fn(f"kblas_{prec.tag}gemv_offset_async")
    if max(m, n, lda, off_r, off_c) > INT_MAX:
        c_int_dims("gemv", m=m, n=n, lda=lda, offset_r=off_r, offset_c=off_c)
    with _on_device(device):
        rc = f(trans.encode(), m, n, _lib.scalar(prec.tag, alpha), a_ptr, lda, x.data_ptr(), 1,
               _lib.scalar(prec.tag, beta), y.data_ptr(), 1, off_r, off_c, stream_handle(device))
    _lib.check(rc, f"kblas_{prec.tag}gemv_offset",
               ["trans", "m", "n", "alpha", "A", "lda", "x", "incx", "beta", "y", "incy", "offset_r", "offset_c"])


def call_symv(prec: Precision, hermitian: bool, uplo: str, d: int, alpha, a_ptr: int, lda: int,
              x: torch.Tensor, beta, y: torch.Tensor, device, offset: int = 0):
    """offset: the (offset, offset) diagonal position of the d x d operand from a_ptr."""
    name = SYMV_FN[(prec.tag, bool(hermitian))]
    f = _fn(f"kblas_{name}_offset_async")
    if max(d, lda, offset) > INT_MAX:
        c_int_dims(name, n=d, lda=lda, offset=offset)
    with _on_device(device):
        rc = f(uplo.encode(), d, _lib.scalar(prec.tag, alpha), a_ptr, lda, x.data_ptr(), 1,
               _lib.scalar(prec.tag, beta), y.data_ptr(), 1, offset, stream_handle(device))
    _lib.check(rc, f"kblas_{name}_offset",
               ["uplo", "n", "alpha", "A", "lda", "x", "incx", "beta", "y", "incy", "offset"])


def host_vectors(x, y, inplace: bool) -> bool:
    """numpy (host) x and y: the call goes through kblas_mv_hostvec."""
    return not inplace and not _is_torch(x) and not _is_torch(y)


class _PinnedResults:
    """Page-locked result buffers for the numpy-vector path, reused once
    the numpy array handed to the caller (and every view of it) has been
    released, which the array's reference count shows.  torch's caching
    host allocator records and polls a CUDA event per block (~14 us per
    allocation once earlier results are still alive); no event is needed
    here, because kblas_mv_hostvec has synchronised its stream before the
    array is returned, so the GPU no longer touches a buffer the caller can
    see or release."""

    KEEP_BYTES = 32 << 20  # tracked page-locked bytes per (dtype, length) ...
    KEEP_MIN, KEEP_MAX = 8, 64  # ... as 8..64 buffers; beyond that, untracked allocations

    def __init__(self):
        self._bufs: dict = {}
        self._next: dict = {}  # round-robin scan start per key
        self._lock = threading.Lock()
        # reference count of an array held only by its pool entry, measured
        # the way get() measures it (interpreter-version independent)
        probe = [(None, np.zeros(1))]
        self._free_refs = min(self._refs(e) for e in probe)

    @staticmethod
    def _refs(entry) -> int:
        return sys.getrefcount(entry[1])

    def get(self, n: int, dtype: torch.dtype):
        key = (dtype, n)
        with self._lock:
            lst = self._bufs.setdefault(key, [])
            k = len(lst)
            # round robin from the buffer after the last one handed out: with
            # results released in call order (a queue of pending calls) the
            # first candidate is free
            start = self._next.get(key, 0)
            for i in range(k):
                j = (start + i) % k
                entry = lst[j]
                if self._refs(entry) <= self._free_refs:
                    self._next[key] = j + 1
                    # a new tuple: it holds the array (count above free)
                    # before the lock is released
                    return entry[0], entry[1]
            t = torch.empty(n, dtype=dtype, pin_memory=True)
            entry = (t, t.numpy())
            keep = max(self.KEEP_MIN, min(self.KEEP_MAX, self.KEEP_BYTES // max(1, t.numel() * t.element_size())))
            if k < keep:
                lst.append(entry)
                self._next[key] = k + 1
            return entry[0], entry[1]


_PINNED = _PinnedResults()


def _hostvec_operands(prec: Precision, x, x_len: int, alpha, beta, y, y_len: int, placeholder):
    """Slow path of call_hostvec: convert and validate the operands the way
    kernels.py:395-399 does (same exceptions and messages)."""
    xa = np.ascontiguousarray(np.asarray(x, dtype=prec.dtype))
    if xa.ndim != 1 or xa.size != x_len:
        raise ValueError(f"x must be a vector of length {x_len}")
    a_c, b_c = _lib.scalar(prec.tag, alpha), _lib.scalar(prec.tag, beta)
    if prec.is_complex:
        alpha, beta = complex(a_c.re, a_c.im), complex(b_c.re, b_c.im)
    else:
        alpha, beta = float(a_c.value), float(b_c.value)
    if complex(beta) == 0:
        if length_of(y) != y_len:
            raise ValueError(f"y must be a vector of length {y_len}")
        ya = placeholder  # never read: any vector of the right length
    else:
        ya = np.ascontiguousarray(np.asarray(y, dtype=prec.dtype))
        if ya.ndim != 1 or ya.size != y_len:
            raise ValueError(f"y must be a vector of length {y_len}")
    return xa, alpha, beta, ya


_HC_MOD = None


def hostcall():
    """The CPython binding of kblas_mv_hostvec (csrc/kblas_hostcall.cpp,
    built in-tree next to libkblas_b200.so).  Imported on first use so the
    package (and its build module) imports before anything is built; a
    missing binding raises here, there is no other path."""
    global _HC_MOD
    if _HC_MOD is None:
        try:
            from . import _hostcall
        except ImportError as e:
            raise ImportError(
                f"paper_1410_1726_b200/_hostcall is missing or cannot load ({e}): build it with "
                "`python -m paper_1410_1726_b200._build` (there is no CPU fallback)"
            ) from e
        _HC_MOD = _hostcall
    return _HC_MOD


def call_hostvec(prec: Precision, kind: str, op: str, hermitian: bool, m: int, n: int, alpha, a_ptr: int,
                 lda: int, x, x_len: int, beta, y, y_len: int, device, off_r: int = 0, off_c: int = 0,
                 keep: list | None = None):
    """One call of the numpy-vector path through the CPython binding of
    kblas_mv_hostvec[_async] (csrc/kblas_hostcall.cpp): a copy-in grid
    stages x (and y when beta != 0) from page-locked memory, the kernels
    run, the result lands in a page-locked buffer from _PinnedResults, and
    the call waits.  Returns (numpy result, launch plan).

    Operands that are not already 1-D contiguous arrays of the operand
    dtype are converted and validated here first (_hostvec_operands).

    keep is not None: asynchronous (a CommandQueue submission): no wait;
    the operands the copy-in grid and kernels still read are appended to
    `keep`, which the caller holds until its queue synchronises.  The
    result buffer comes from the same pool; it is not handed out again
    while the returned array (held by the queue's handle) is alive."""
    _HC = hostcall()
    out, out_np = _PINNED.get(y_len, prec.torch_dtype)
    sync = keep is None
    herm = 1 if hermitian else 0
    with _on_device(device):
        sh = stream_handle(device)
        rc = _HC.mv_hostvec(prec.tag, kind, op, herm, m, n, alpha, a_ptr, lda, off_r, off_c, x, x_len, beta, y,
                            y_len, out.data_ptr(), sh, sync)
        if rc == _HC.SLOW_PATH:
            x, alpha, beta, y = _hostvec_operands(prec, x, x_len, alpha, beta, y, y_len, out_np)
            rc = _HC.mv_hostvec(prec.tag, kind, op, herm, m, n, alpha, a_ptr, lda, off_r, off_c, x, x_len, beta,
                                y, y_len, out.data_ptr(), sh, sync)
            if rc == _HC.SLOW_PATH:
                raise RuntimeError("kblas_mv_hostvec: converted operands rejected by the fast path")
    _lib.check(rc, "kblas_mv_hostvec" if sync else "kblas_mv_hostvec_async")
    if keep is not None:
        keep.extend((x, y, out))
    return out_np, _HC.last_plan()
