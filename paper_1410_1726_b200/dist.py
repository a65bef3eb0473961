"""One-process-per-GPU mgpu path (torchrun / torch.distributed).

Same 1D block-column-cyclic layout as multidevice.py (multidevice.py:1-9):
rank r owns block columns j = r, r + G, ... of width nb and stores them
packed in a local panel.  Each rank computes its partial y with the sm_100a
kernels (`partial_mv`), then the exchange step — the one real collective
of the path — is an NCCL reduce(sum) of the partials onto rank 0, where
beta*y is added (multidevice.py:276,282-283).  GEMV-T partials have
disjoint support, so the same reduce is exact for them.

The partial computation is injectable so the orchestration is covered by
world_size-2 gloo tests on CPU (tests/test_dist_gloo.py).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .multidevice import local_col_count, local_ld, owned_block_cols


def owned_columns(n: int, nb: int, world: int, rank: int) -> np.ndarray:
    """Global column indices of rank's panel, in local order."""
    blocks = owned_block_cols(n, nb, world, rank)
    if not blocks:
        return np.zeros(0, dtype=np.int64)
    return np.concatenate([np.arange(j * nb, min(n, (j + 1) * nb)) for j in blocks])


def panel_shape(m: int, n: int, nb: int, world: int, rank: int) -> tuple[int, int, int]:
    """(rows, local columns, ld) of rank's panel (multidevice.py:46-52)."""
    return m, local_col_count(n, nb, world, rank), local_ld(m)


def combine(partial: torch.Tensor, y: torch.Tensor | None, beta, group=None) -> torch.Tensor | None:
    """Sum the ranks' partials onto rank 0 and add beta*y there.

    Returns the result on rank 0 and None elsewhere.  `partial` is consumed
    (used as the reduce buffer)."""
    dist.reduce(partial, dst=0, op=dist.ReduceOp.SUM, group=group)
    if dist.get_rank(group) != 0:
        return None
    if complex(beta) == 0:
        return partial
    return y * torch.as_tensor(beta, dtype=y.dtype, device=y.device) + partial


def mv_dist(kind: str, op: str, m: int, n: int, alpha, panel, x: torch.Tensor, beta, y, nb: int,
            partial_fn, group=None, hermitian: bool = False):
    """Distributed y = alpha * op(A) x + beta * y over `group`.

    partial_fn(kind, op, m, n, alpha, panel, x, out, world, rank, nb, hermitian)
    fills `out` with this rank's alpha-scaled partial."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    y_len = m if (kind == "g" and op == "n") else n
    out = torch.empty(y_len, dtype=x.dtype, device=x.device)
    partial_fn(kind, op, m, n, alpha, panel, x, out, world, rank, nb, hermitian)
    return combine(out, y, beta, group)


def gpu_partial(prec):
    """partial_fn backed by the sm_100a library (kblas_mv_mgpu_partial_async)."""
    from .multidevice import partial_mv

    def fn(kind, op, m, n, alpha, panel, x, out, world, rank, nb, hermitian):
        partial_mv(prec, kind, op, m, n, alpha, panel, x, out, world, rank, nb, hermitian)

    return fn


class P2PExchange:
    """Peer-memory exchange of the per-rank partials (no NCCL on the data
    path): the root (rank 0) owns a slot per rank plus flags in HBM and
    shares them with CUDA IPC.  Each rank's partial goes straight into its
    slot (NVLink stores when ranks are on different GPUs) and its arrival
    is published with a system-scope release; the root sums the slots in
    rank order with beta*y (multidevice.py:276,282-283: the device-order
    sum, so the result does not depend on arrival order) and releases the
    slots for the next call.  For SYMV/HEMV all of this happens inside the
    partial's epilogue kernel.  Synchronisation is on the device; the
    process group is used once, to exchange the IPC handles.  One call:
    `p2p_mv(..., ex)`."""

    def __init__(self, n: int, dtype: torch.dtype, group=None):
        import ctypes

        from . import _lib
        from ._ops import stream_handle

        self._lib = _lib.load()
        self._stream = stream_handle
        self.group = group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.n, self.dtype = n, dtype
        self.dev = torch.device("cuda", torch.cuda.current_device())
        esize = torch.empty(0, dtype=dtype).element_size()
        self.ld = -(-n * esize // 256) * 256 // esize  # 256-byte aligned slots
        self.seq = 0
        # every rank learns whether every rank could map the slots, so a
        # failure on one rank raises on all of them (a rank left on the p2p
        # path would otherwise wait for peers that took another path)
        err = None
        payload = [None]
        if self.rank == 0:
            try:
                self._slots = torch.zeros(self.world * self.ld, dtype=dtype, device=self.dev)
                self._ctl = torch.zeros(self.world + 2, dtype=torch.int64, device=self.dev)  # flags, consumed, counter
                handles = []
                for t in (self._slots, self._ctl):
                    h = (ctypes.c_char * 64)()
                    _lib.check(self._lib.kblas_ipc_get_handle(t.data_ptr(), h), "kblas_ipc_get_handle")
                    # the allocation may start before the tensor (caching allocator)
                    handles.append((bytes(h), t.data_ptr() - self._base_of(t)))
                payload = [handles]
            except Exception as e:  # noqa: BLE001 - reported on every rank below
                err = f"rank 0: {e}"
                payload = [err]
        dist.broadcast_object_list(payload, src=0, group=group)
        self._opened = []
        ptrs = []
        if isinstance(payload[0], str):
            err = payload[0]
        elif self.rank != 0:
            try:
                for h, off in payload[0]:
                    p = ctypes.c_void_p()
                    _lib.check(self._lib.kblas_ipc_open_handle(h, ctypes.byref(p)), "kblas_ipc_open_handle")
                    self._opened.append(p.value)
                    ptrs.append(p.value + off)
            except Exception as e:  # noqa: BLE001
                err = f"rank {self.rank}: {e}"
        ok = self._agree(err is None, group)
        if not ok:
            self.close()
            raise RuntimeError(f"p2p exchange unavailable on some rank ({err or 'another rank failed'})")
        if self.rank == 0:
            self.slots_ptr, ctl_ptr = self._slots.data_ptr(), self._ctl.data_ptr()
        else:
            self.slots_ptr, ctl_ptr = ptrs
        self.flags_ptr = ctl_ptr
        self.consumed_ptr = ctl_ptr + 8 * self.world
        self.counter_ptr = ctl_ptr + 8 * (self.world + 1)
        self._esize = esize

    @staticmethod
    def _agree(ok: bool, group) -> bool:
        """True on every rank iff ok on every rank (one MIN all-reduce)."""
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        return bool(t.item())

    @staticmethod
    def _base_of(t: torch.Tensor) -> int:
        """Start of the cudaMalloc block holding t (what an IPC handle names)."""
        import ctypes

        base = ctypes.c_void_p()
        size = ctypes.c_size_t()
        lib = ctypes.CDLL("libcuda.so.1")
        rc = lib.cuMemGetAddressRange_v2(ctypes.byref(base), ctypes.byref(size), ctypes.c_void_p(t.data_ptr()))
        if rc != 0:
            raise RuntimeError(f"cuMemGetAddressRange failed ({rc})")
        return base.value

    def close(self):
        for p in self._opened:
            self._lib.kblas_ipc_close(p)
        self._opened = []


def p2p_mv(prec, kind: str, op: str, m: int, n: int, alpha, panel, x: torch.Tensor, beta, y, nb: int,
           ex: P2PExchange, hermitian: bool = False):
    """Distributed y = alpha * op(A) x + beta * y with the peer-memory
    exchange (kblas_mv_mgpu_partial_p2p_async): this rank's partial goes
    into its slot in rank 0's HBM, rank 0 adds the slots in rank order with
    beta*y.  For SYMV/HEMV the exchange runs inside the partial's epilogue
    kernel.  Returns the result on rank 0, None elsewhere."""
    import ctypes

    from . import _lib, _ops
    from ._ops import stream_handle

    lib = _lib.load()
    a_ptr, lda = (0, 1)
    if panel is not None:
        a_ptr = panel.data.data_ptr() + panel.linear_index(0, 0) * prec.element_bytes
        lda = panel.ld
    ex.seq += 1
    plen = m if (kind == "g" and op == "n") else n
    root = ex.rank == 0
    out = torch.empty(plen, dtype=x.dtype, device=x.device) if root else None
    bz = complex(beta) == 0
    if root and not bz:
        if y is None or y.numel() != plen:
            raise ValueError(f"y must be a vector of length {plen}")
        y = y.to(device=x.device, dtype=x.dtype).contiguous()
    al, be = _lib.scalar(prec.tag, alpha), _lib.scalar(prec.tag, beta)
    _ops.c_int_dims("mgpu p2p partial", m=m, n=n, lda=lda)
    rc = lib.kblas_mv_mgpu_partial_p2p_async(
        prec.tag.encode(), kind.encode(), op.encode(), m, n, ctypes.addressof(al), a_ptr, lda, x.data_ptr(),
        ex.world, ex.rank, nb, 1 if hermitian else 0, ex.slots_ptr, ex.ld, ex.flags_ptr, ex.consumed_ptr,
        ex.counter_ptr, ex.seq, ctypes.addressof(be), y.data_ptr() if (root and not bz) else None,
        out.data_ptr() if root else None, stream_handle(x.device))
    _lib.check(rc, "kblas_mv_mgpu_partial_p2p_async")
    return out
