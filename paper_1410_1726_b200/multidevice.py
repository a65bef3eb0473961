"""1D block-column-cyclic multi-GPU GEMV / SYMV / HEMV (multidevice.py:1-332).

Layout: block column j of width nb lives on GPU j mod G,
packed contiguously into that GPU's local panel whose ld is the row count
padded to 32 elements (multidevice.py:72-93).  Each GPU runs the same
sm_100a kernels on its panel: a column map turns local columns into
global ones, so GEMV-N and SYMV/HEMV produce a full-length partial y and
GEMV-T produces its own disjoint segments (zeros elsewhere).  Partials are
then combined on the root GPU, by library kernels only:

  reduce="ordered" (default): one `kblas_x*_mgpu_async` call -- every
      GPU's partial on its own stream, then a root kernel that reads the
      partials in device order over NVLink peer memory and fuses beta*y
      (multidevice.py:161,176,276,282-283), so results are deterministic;
  reduce="nccl": the per-GPU partial kernels, one `ncclReduce(sum)` onto
      the root (torch.cuda.nccl, the torch-bundled NCCL), then the root
      combine kernel (`kblas_mv_mgpu_combine_async`) for beta*y.

The x copies and the non-root partial buffers are cached per device and
reused across calls (stream-ordered: every GPU's stream waits for the
root's combine before the next partial overwrites its buffer).

Logical GPUs may share a physical device (e.g. G=8 on a 1-GPU box maps
every logical GPU to cuda:0); the math is identical, only the placement
changes.  For one-process-per-GPU deployments see `partial_mv` and
bench.py, which reduce partials with torch.distributed (NCCL).

`CommandQueue` keeps the reference contract (multidevice.py:287-332): work
is enqueued in submission order, `result()` before `synchronize()` raises
RuntimeError("queue not synchronized yet").  On B200 submission launches
immediately on the queue's own CUDA stream; synchronize waits for it.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, _ops
from .core import WARP_SIZE, MatrixView, Precision, _is_torch, alloc_matrix
from .kernels import ExecutionReport, _is_one, _is_zero
from .partition import DEFAULT_CONFIG, KernelConfig


def block_col_count(n: int, nb_cols: int) -> int:
    return -(-n // nb_cols)


def owned_block_cols(n: int, nb_cols: int, device_count: int, device: int) -> list[int]:
    """Block columns of one GPU (multidevice.py:33-35)."""
    return list(range(device, block_col_count(n, nb_cols), device_count))


def local_col_count(n: int, nb_cols: int, device_count: int, device: int) -> int:
    """Columns held by one GPU, tail block included (multidevice.py:38-43)."""
    total = 0
    for j in owned_block_cols(n, nb_cols, device_count, device):
        total += min(n, (j + 1) * nb_cols) - j * nb_cols
    return total


def local_ld(m: int) -> int:
    return -(-m // WARP_SIZE) * WARP_SIZE


def required_local_elements(m: int, n: int, nb_cols: int, device_count: int, device: int) -> int:
    """Allocation size of one GPU's panel (multidevice.py:46-52)."""
    cols = local_col_count(n, nb_cols, device_count, device)
    return 0 if cols == 0 else local_ld(m) * cols


def default_devices(device_count: int) -> list[torch.device]:
    _ops.require_cuda()
    phys = torch.cuda.device_count()
    return [torch.device("cuda", g % phys) for g in range(device_count)]


@dataclass
class DistributedMatrix:
    global_m: int
    global_n: int
    nb_cols: int
    device_count: int
    precision: Precision
    local_views: list  # MatrixView | None per logical GPU
    devices: list = field(default_factory=list)

    @property
    def block_cols(self) -> int:
        return block_col_count(self.global_n, self.nb_cols)

    def owned(self, device: int) -> list[int]:
        return owned_block_cols(self.global_n, self.nb_cols, self.device_count, device)


def _as_torch_2d(view: MatrixView):
    a = view.array()
    return a if _is_torch(a) else torch.from_numpy(a)


def distribute(a: MatrixView, nb_cols: int, device_count: int, devices=None) -> DistributedMatrix:
    """Pack block columns cyclically onto the GPUs (multidevice.py:72-93)."""
    if device_count < 1 or nb_cols < 1:
        raise ValueError("device_count and nb_cols must be >= 1")
    devices = [torch.device(d) for d in devices] if devices is not None else default_devices(device_count)
    if len(devices) != device_count:
        raise ValueError("need one device per logical GPU")
    m, n = a.rows, a.cols
    src = _as_torch_2d(a)
    locals_ = []
    for g in range(device_count):
        owned = owned_block_cols(n, nb_cols, device_count, g)
        if not owned:
            locals_.append(None)  # idle GPU (multidevice.py:81-83)
            continue
        width = local_col_count(n, nb_cols, device_count, g)
        local = alloc_matrix(m, width, a.precision, ld=local_ld(m), device=devices[g])
        dst = local.array()
        pos = 0
        for j in owned:
            c0, c1 = j * nb_cols, min(n, (j + 1) * nb_cols)
            dst[:, pos:pos + (c1 - c0)].copy_(src[:, c0:c1], non_blocking=True)
            pos += c1 - c0
        locals_.append(local)
    return DistributedMatrix(m, n, nb_cols, device_count, a.precision, locals_, devices)


def gather(dist: DistributedMatrix, device=None) -> MatrixView:
    """Reassemble the global matrix (multidevice.py:96-110) on `device`
    (default: the first GPU; "numpy" for a host copy)."""
    dev = device if device is not None else dist.devices[0]
    out = alloc_matrix(dist.global_m, dist.global_n, dist.precision, ld=dist.global_m, device=dev)
    dst = _as_torch_2d(out)
    for g in range(dist.device_count):
        local = dist.local_views[g]
        if local is None:
            continue
        src = local.array()
        pos = 0
        for j in dist.owned(g):
            c0, c1 = j * dist.nb_cols, min(dist.global_n, (j + 1) * dist.nb_cols)
            dst[:, c0:c1].copy_(src[:, pos:pos + (c1 - c0)])
            pos += c1 - c0
    return out


# --------------------------------------------------------------------------
# per-GPU partial (the building block; also used by one-process-per-GPU runs)
# --------------------------------------------------------------------------
def partial_mv(prec: Precision, kind: str, op: str, m: int, n: int, alpha, local: MatrixView | None,
               x: torch.Tensor, out: torch.Tensor, device_count: int, device_index: int, nb: int,
               hermitian: bool = False):
    """out = alpha * (contribution of logical GPU `device_index`) on out's device.

    kind 'g' (gemv, op n/t/c, out length m for 'n' else n) or 's'
    (symv/hemv, op l/u, out length n).  local None -> zero partial."""
    lib = _lib.load()
    dev = out.device
    a_ptr, lda = (0, 1)
    if local is not None:
        a_ptr = local.data.data_ptr() + local.linear_index(0, 0) * prec.element_bytes
        lda = local.ld
    al = _lib.scalar(prec.tag, alpha)
    _ops.c_int_dims("mgpu partial", m=m, n=n, lda=lda)
    with _ops._on_device(dev):
        rc = lib.kblas_mv_mgpu_partial_async(
            prec.tag.encode(), kind.encode(), op.encode(), m, n, ctypes.cast(ctypes.byref(al), ctypes.c_void_p),
            a_ptr, lda, x.data_ptr(), out.data_ptr(), device_count, device_index, nb, 1 if hermitian else 0,
            _ops.stream_handle(dev))
    _lib.check(rc, "kblas_mv_mgpu_partial_async")


_scratch: dict = {}


def _buffer(dev: torch.device, dtype: torch.dtype, n: int, role) -> torch.Tensor:
    """A cached length-n device vector (x copies, non-root partials): reused
    across calls, ordered by the streams (see the module docstring)."""
    key = (dev.index, dtype, role)
    t = _scratch.get(key)
    if t is None or t.numel() < n:
        t = torch.empty(n, dtype=dtype, device=dev)
        _scratch[key] = t
    return t[:n]


def _mgpu_name(prec: Precision, kind: str, hermitian: bool) -> str:
    if kind == "g":
        return f"{prec.tag}gemv"
    return {"s": "ssymv", "d": "dsymv", "c": "chemv" if hermitian else "csymv",
            "z": "zhemv" if hermitian else "zsymv"}[prec.tag]


def _ptr_array(vals):
    return (ctypes.c_void_p * len(vals))(*[v if v else None for v in vals])


def _mgpu_common(kind: str, op: str, alpha, dist: DistributedMatrix, x, beta, y, x_len: int, y_len: int,
                 hermitian: bool, reduce: str):
    prec = dist.precision
    root = dist.devices[0]
    G = dist.device_count
    lib = _lib.load()
    xd = _ops.vector_in(x, x_len, prec, "x", root)
    yd = _ops.vector_in(y, y_len, prec, "y", root)
    bz = _is_zero(beta)
    # dy[0]: y on input, the result on output (a fresh vector, as in the reference)
    out = torch.empty_like(yd) if bz else yd.clone()
    # x on every physical device (one cached copy per device)
    xs = {}
    for dev in dist.devices:
        if dev.index in xs:
            continue
        if dev == root:
            xs[dev.index] = xd
        else:
            with _ops._on_device(dev):
                xs[dev.index] = _buffer(dev, prec.torch_dtype, x_len, "x").copy_(xd, non_blocking=True)
    eb = prec.element_bytes
    a_ptrs = [(v.data.data_ptr() + v.linear_index(0, 0) * eb) if v is not None else 0 for v in dist.local_views]
    lda = next((v.ld for v in dist.local_views if v is not None), local_ld(dist.global_m))
    _ops.c_int_dims("mgpu", m=dist.global_m, n=dist.global_n, lda=lda)
    streams = [_ops.stream_handle(dev) for dev in dist.devices]
    distinct = len({d.index for d in dist.devices}) == G
    al, be = _lib.scalar(prec.tag, alpha), _lib.scalar(prec.tag, beta)
    if reduce == "nccl" and G > 1 and distinct and not _is_zero(alpha):
        # per-GPU partials, NCCL reduce(sum) onto the root, root combine with beta
        parts = [_buffer(dev, prec.torch_dtype, y_len, ("part", g)) for g, dev in enumerate(dist.devices)]
        for g, dev in enumerate(dist.devices):
            partial_mv(prec, kind, op, dist.global_m, dist.global_n, alpha, dist.local_views[g], xs[dev.index],
                       parts[g], G, g, dist.nb_cols, hermitian)
        torch.cuda.nccl.reduce(parts, output=parts[0], root=0)
        with _ops._on_device(root):
            rc = lib.kblas_mv_mgpu_combine_async(prec.tag.encode(), y_len, 1, _ptr_array([parts[0].data_ptr()]),
                                                 ctypes.addressof(be), out.data_ptr(), streams[0])
        _lib.check(rc, "kblas_mv_mgpu_combine_async")
        return out
    dys = [out.data_ptr()] + [_buffer(dist.devices[g], prec.torch_dtype, y_len, ("part", g)).data_ptr()
                              for g in range(1, G)]
    ids = (ctypes.c_int * G)(*[d.index for d in dist.devices])
    sts = (ctypes.c_void_p * G)(*streams)
    name = f"kblas_{_mgpu_name(prec, kind, hermitian)}_mgpu_async"
    args = [_ptr_array(a_ptrs), lda, _ptr_array([xs[d.index].data_ptr() for d in dist.devices]), 1, be,
            _ptr_array(dys), 1, G, dist.nb_cols, ids, sts]
    with _ops._on_device(root):
        if kind == "g":
            rc = getattr(lib, name)(op.encode(), dist.global_m, dist.global_n, al, *args)
        else:
            rc = getattr(lib, name)(op.encode(), dist.global_n, al, *args)
    _lib.check(rc, name)
    return out


def _device_reports(dist: DistributedMatrix, kind: str, trans_or_uplo: str, alpha) -> list:
    prec = dist.precision
    mul, add, eb = prec.flops_per_mul, prec.flops_per_add, prec.element_bytes
    m, n, nb = dist.global_m, dist.global_n, dist.nb_cols
    reps = []
    for g in range(dist.device_count):
        rep = ExecutionReport()
        local = dist.local_views[g]
        if local is not None and not _is_zero(alpha):
            lc = local.cols
            if kind == "g":
                if trans_or_uplo == "n":
                    rep.flops = mul * (m * lc + m) + add * (m * lc)  # multidevice.py:171-172
                    elems, xl, yl = m * lc, lc, m
                else:
                    rep.flops = mul * (lc * m + lc) + add * (lc * m)
                    elems, xl, yl = m * lc, m, lc
            else:
                elems = 0
                for j in dist.owned(g):
                    c0, c1 = j * nb, min(n, (j + 1) * nb)
                    pw = c1 - c0
                    off_rows = (n - c1) if trans_or_uplo == "l" else c0
                    rep.flops += mul * (pw * pw + pw) + add * pw * pw  # diagonal (multidevice.py:248-250)
                    rep.flops += 2 * (mul + add) * off_rows * pw       # off-diagonal (multidevice.py:269-270)
                    elems += pw * (pw + 1) // 2 + off_rows * pw
                xl, yl = n, n
            rep.matrix_transactions = -(-elems * eb // 128)
            rep.bytes_read = (elems + xl) * eb
            rep.bytes_written = yl * eb
            rep.transactions = rep.matrix_transactions + -(-(xl + yl) * eb // 128)
            rep.tb_count = 1
        reps.append(rep)
    return reps


def _merge(reps: list, y_out) -> ExecutionReport:
    merged = ExecutionReport()
    for r in reps:
        merged.absorb(r)
    merged.y_out = y_out
    return merged


def gemv_mgpu(trans: str, alpha, dist: DistributedMatrix, x, beta, y, config: KernelConfig = DEFAULT_CONFIG,
              reduce: str = "ordered"):
    """General MV over a distributed matrix (multidevice.py:119-180).
    Returns (merged_report, per_device_reports)."""
    trans = trans.lower()
    if trans not in ("n", "t", "c"):
        raise ValueError(f"trans must be 'n', 't' or 'c', got {trans!r}")
    prec = dist.precision
    if trans == "c" and not prec.is_complex:
        trans = "t"
    m, n = dist.global_m, dist.global_n
    x_len, y_len = (n, m) if trans == "n" else (m, n)
    for v, L in ((x, x_len), (y, y_len)):
        if (v.numel() if _is_torch(v) else np.asarray(v).size) != L:
            raise ValueError(f"expected x of length {x_len} and y of length {y_len}")
    out = _mgpu_common("g", trans, alpha, dist, x, beta, y, x_len, y_len, False, reduce)
    per = _device_reports(dist, "g", trans, alpha)
    return _merge(per, _ops.result_like(y, out)), per


def symv_hemv_mgpu(uplo: str, alpha, dist: DistributedMatrix, x, beta, y, config: KernelConfig = DEFAULT_CONFIG,
                   hermitian: bool | None = None, reduce: str = "ordered"):
    """Symmetric/Hermitian MV over a triangle-stored distributed matrix
    (multidevice.py:183-284).  Returns (merged_report, per_device_reports)."""
    uplo = uplo.lower()
    if uplo not in ("l", "u"):
        raise ValueError(f"uplo must be 'l' or 'u', got {uplo!r}")
    if dist.global_m != dist.global_n:
        raise ValueError("symmetric ops need a square distributed matrix")
    if dist.nb_cols != config.block_size:
        raise ValueError("distribution block width must equal the kernel block size for symmetric ops")
    prec = dist.precision
    if hermitian is None:
        hermitian = prec.is_complex
    if hermitian and not prec.is_complex:
        raise ValueError("hermitian treatment requires a complex precision")
    d = dist.global_n
    for v in (x, y):
        if (v.numel() if _is_torch(v) else np.asarray(v).size) != d:
            raise ValueError(f"expected x and y of length {d}")
    out = _mgpu_common("s", uplo, alpha, dist, x, beta, y, d, d, hermitian, reduce)
    per = _device_reports(dist, "s", uplo, alpha)
    return _merge(per, _ops.result_like(y, out)), per


class CommandQueue:
    """In-order queue with the reference contract (multidevice.py:287-303).

    Submitted work is launched at once on this queue's CUDA stream (one per
    device it touches is not needed: cross-device work is ordered with
    events inside the mgpu calls); `synchronize()` waits for the stream and
    releases the handles' results."""

    def __init__(self, name: str = "default", device=None):
        self.name = name
        self._pending: list = []
        self._stream = None
        self._device = device

    @property
    def stream(self):
        if self._stream is None and torch.cuda.is_available():
            dev = self._device if self._device is not None else torch.cuda.current_device()
            self._stream = torch.cuda.Stream(device=dev)
        return self._stream

    def submit(self, fn, *args, **kwargs) -> "_Pending":
        handle = _Pending(self, fn, args, kwargs)
        st = self.stream
        if st is None:
            handle._run()
        elif st.device_index == torch._C._cuda_getDevice():
            # fast path (the queue lives on the current device): order the
            # queue after the caller's stream with one event on the device
            # and swap torch's current stream directly (torch.cuda.stream()
            # and wait_stream() cost ~20 us of Python per submission)
            idx = st.device_index
            _lib.check(_ops._fn("kblas_stream_order")(st.cuda_stream, _ops.stream_handle(idx)),
                       "kblas_stream_order")
            prev = torch._C._cuda_getCurrentStream(idx)
            torch._C._cuda_setStream(stream_id=st.stream_id, device_index=idx, device_type=st.device_type)
            try:
                handle._run()
            finally:
                torch._C._cuda_setStream(stream_id=prev[0], device_index=prev[1], device_type=prev[2])
        else:
            st.wait_stream(torch.cuda.current_stream(st.device))
            with torch.cuda.stream(st):
                handle._run()
        self._pending.append(handle)
        return handle

    def synchronize(self) -> None:
        if self._stream is not None:
            self._stream.synchronize()
        pending, self._pending = self._pending, []
        for h in pending:
            h.done = True


@dataclass
class _Pending:
    queue: CommandQueue
    fn: object
    args: tuple
    kwargs: dict
    done: bool = False
    _result: object = field(default=None, repr=False)

    def _run(self):
        self._result = self.fn(*self.args, **self.kwargs)

    def result(self):
        if not self.done:
            raise RuntimeError("queue not synchronized yet")
        return self._result


def gemv_mgpu_async(trans, alpha, dist, x, beta, y, config, queue: CommandQueue) -> _Pending:
    return queue.submit(gemv_mgpu, trans, alpha, dist, x, beta, y, config)


def symv_hemv_mgpu_async(uplo, alpha, dist, x, beta, y, config, queue: CommandQueue, hermitian=None) -> _Pending:
    return queue.submit(symv_hemv_mgpu, uplo, alpha, dist, x, beta, y, config, hermitian)
