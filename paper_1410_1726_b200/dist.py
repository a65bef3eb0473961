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
