"""World-size-2 gloo test of the one-process-per-GPU mgpu orchestration
(paper_1410_1726_b200/dist.py): block-cyclic ownership, per-rank partials,
the reduce onto rank 0 and the beta fusion.  The per-rank partial here is a
CPU stand-in (numpy on the rank's owned columns) because this container
has no GPU; on the B200 the same orchestration runs with gpu_partial()
and NCCL (bench.py --gpus N)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1410_1726_b200.dist import mv_dist, owned_columns, panel_shape


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def cpu_partial(kind, op, m, n, alpha, panel, x, out, world, rank, nb, hermitian):
    """alpha * (rank's contribution), numpy restatement of multidevice.py:224-276."""
    A = panel  # global dense matrix (test stand-in for the rank's panel)
    cols = owned_columns(n, nb, world, rank)
    xs = x.numpy()
    if kind == "g":
        if op == "n":
            res = A[:, cols] @ xs[cols]
        else:
            res = np.zeros(n, dtype=A.dtype)
            res[cols] = A[:, cols].T @ xs
    else:
        tri = np.tril(A) if op == "l" else np.triu(A)
        strict = np.tril(A, -1) if op == "l" else np.triu(A, 1)
        res = np.zeros(n, dtype=A.dtype)
        res += tri[:, cols] @ xs[cols]          # stored elements of owned columns -> rows
        res[cols] += strict[:, cols].T @ xs      # mirrored products -> owned columns
    out.copy_(torch.from_numpy(alpha * res))


def _worker(rank, world, port, kind, op, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(5)
    n, nb = 300, 32
    A = rng.uniform(-1, 1, (n, n))
    x = torch.from_numpy(rng.uniform(-1, 1, n))
    y = torch.from_numpy(rng.uniform(-1, 1, n))
    res = mv_dist(kind, op, n, n, 0.7, A, x, -1.5, y, nb, cpu_partial)
    if rank == 0:
        if kind == "g":
            want = 0.7 * ((A if op == "n" else A.T) @ x.numpy()) - 1.5 * y.numpy()
        else:
            full = np.tril(A) + np.tril(A, -1).T if op == "l" else np.triu(A) + np.triu(A, 1).T
            want = 0.7 * (full @ x.numpy()) - 1.5 * y.numpy()
        q.put(float(np.max(np.abs(res.numpy() - want))))
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,op", [("g", "n"), ("g", "t"), ("s", "l"), ("s", "u")])
def test_mv_dist_world2(kind, op):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, op, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=5) < 1e-10


def test_ownership_partition_and_panels():
    for n, nb in ((1000, 128), (333, 32), (100000, 128)):
        for world in (1, 2, 3, 8):
            cols = np.concatenate([owned_columns(n, nb, world, r) for r in range(world)])
            assert np.array_equal(np.sort(cols), np.arange(n))
            assert sum(panel_shape(n, n, nb, world, r)[1] for r in range(world)) == n
