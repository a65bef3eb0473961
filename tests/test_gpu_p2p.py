"""The peer-memory exchange of the one-process-per-GPU mgpu path
(dist.P2PExchange / p2p_mv): world size 2, rank r on cuda:(r % #GPUs) —
two processes on one B200 here, two GPUs (cross-device IPC mapping,
NVLink stores, system-scope flags) on a multi-GPU box.  gloo carries the
one-time IPC handle exchange; the data path is CUDA IPC peer stores plus
device flags, no NCCL.  Several calls in a row check the
slot reuse handshake; rank 0's result must match the single-GPU API."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, kind, op, tag, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1410_1726_b200 as kb
    from oracle import gen
    from paper_1410_1726_b200.dist import P2PExchange, p2p_mv

    prec = kb.precision(tag)
    n, nb = 1000, 64
    # identical operands on every rank's device (counter-based generator)
    A = torch.empty(n, n, dtype=prec.torch_dtype, device=dev)
    gen.fill_columns(A, tag, 3, n, n)
    full = kb.view_of(A.T)  # column-major n x n
    dist_mat = kb.distribute(full, nb, world, devices=[dev] * world)
    panel = dist_mat.local_views[rank]
    herm = kind == "s" and prec.is_complex
    ex = P2PExchange(n, prec.torch_dtype)
    errs = []
    for it in range(4):
        x = gen.vector_torch(tag, n, 10 + it, dev)
        y = gen.vector_torch(tag, n, 20 + it, dev)
        beta = 0.0 if it % 2 == 0 else -0.5
        res = p2p_mv(prec, kind, op, n, n, 0.75, panel, x, beta, y, nb, ex, hermitian=herm)
        if rank == 0:
            if kind == "g":
                want = kb.gemv(op, 0.75, full, x, beta, y).y_out
            else:
                want = kb.symv_hemv(op, 0.75, kb.HermitianView(full, op), x, beta, y, hermitian=herm).y_out
            torch.cuda.synchronize()
            errs.append(float((res - want).abs().max() / want.abs().max()))
        else:
            assert res is None
    torch.cuda.synchronize()
    dist.barrier()
    ex.close()
    if rank == 0:
        q.put(max(errs))
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,op,tag", [("s", "l", "d"), ("s", "u", "z"), ("g", "n", "d"), ("g", "t", "s")])
def test_p2p_exchange_world2_one_gpu(kind, op, tag):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, op, tag, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    tol = 1e-5 if tag in "sc" else 1e-12
    assert q.get(timeout=5) < tol


@pytest.mark.parametrize("kind,op,tag", [("s", "l", "d"), ("g", "n", "z")])
def test_p2p_exchange_world4_one_gpu(kind, op, tag):
    """Four ranks (the SCALE run's N=4 shape): the root sums three peers'
    slots in rank order and releases them for the next call."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 4, port, kind, op, tag, q)) for r in range(4)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    assert q.get(timeout=5) < 1e-12


def _fail_worker(rank, world, port, failing, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(torch.device("cuda", rank % torch.cuda.device_count()))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1410_1726_b200 import _lib
    from paper_1410_1726_b200.dist import P2PExchange

    if rank == failing:
        lib = _lib.load()

        class _Broken:  # this rank cannot map the root's allocations
            def __getattr__(self, name):
                if name in ("kblas_ipc_open_handle", "kblas_ipc_get_handle"):
                    return lambda *a: 1  # cudaErrorInvalidValue
                return getattr(lib, name)

        _lib.load = lambda: _Broken()
    try:
        P2PExchange(1000, torch.float64)
        q.put((rank, "constructed"))
    except RuntimeError as e:
        q.put((rank, str(e)))
    dist.barrier()  # every rank got here: nobody is left waiting on the exchange
    dist.destroy_process_group()


@pytest.mark.parametrize("failing", [0, 1])
def test_p2p_exchange_failure_raises_on_every_rank(failing):
    """A rank that cannot set up the IPC mapping (here: rank `failing`'s
    handle calls fail) makes the constructor raise on EVERY rank, so the
    ranks agree on the fallback instead of one waiting on the others."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fail_worker, args=(r, 2, port, failing, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = dict(q.get(timeout=5) for _ in range(2))
    assert set(got) == {0, 1}
    for r, msg in got.items():
        assert "p2p exchange unavailable" in msg, (r, msg)
    assert f"rank {failing}" in got[failing]
