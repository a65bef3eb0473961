"""Back-to-back dependent calls on one stream: every main kernel is a
programmatic dependent of the stream's previous kernel (launch_main,
KBLAS_PDL_CHAIN), and every library kernel releases its dependents early,
so each call must wait in griddepcontrol.wait before it reads the previous
call's output.  A chain where each call's x is the previous call's y, over
every kernel form (row-owning / split / stream-K GEMV-N, column-owning /
stream-K GEMV-T, the 1- and 2-CTA/SM SYMV kernels with and without the
split tail grid), must give exactly the results of the same calls
separated by device synchronisations."""

import numpy as np
import pytest
import torch

import paper_1410_1726_b200 as kb

pytestmark = pytest.mark.gpu


def _mat(g, m, n, dtype=torch.float64):
    t = torch.empty(n, m, dtype=dtype, device="cuda").uniform_(-1, 1, generator=g)
    return kb.view_of(t.T)  # column-major m x n


def _chain(ops, x0, sync):
    """Run ops back to back; no other kernel is launched between two
    library calls (outputs are pre-allocated torch.empty buffers, which
    launch nothing), so each call is a programmatic dependent of the
    previous call's last kernel."""
    x = x0
    outs = []
    for f in ops:
        x = f(x)
        outs.append(x)
        if sync:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    return outs


@pytest.mark.parametrize("n", [2048, 4096, 20000])
def test_dependent_chain_equals_synchronised(n):
    g = torch.Generator(device="cuda").manual_seed(n)
    sq = _mat(g, n, n)
    hv = kb.HermitianView(sq, "l")
    tall = _mat(g, n, 64)   # GEMV-T of a tall panel (column-owning or stream-K)
    wide = _mat(g, 64, n)   # GEMV-N of a short-wide panel (split forms)
    a = 1.7 / n ** 0.5      # keeps the vector norm about constant along the chain

    def new(k):
        return torch.empty(k, dtype=torch.float64, device="cuda")

    def symv(x):
        return kb.symv_hemv("l", a, hv, x, 0.0, new(n), inplace=True).y_out

    def gemv_n(x):
        return kb.gemv("n", a, sq, x, 0.0, new(n), inplace=True).y_out

    def gemv_t(x):
        return kb.gemv("t", a, sq, x, 0.0, new(n), inplace=True).y_out

    def through_panels(x):
        t = kb.gemv("t", a, tall, x, 0.0, new(64), inplace=True).y_out
        return kb.gemv("t", 1.0 / 8, wide, t, 0.0, new(n), inplace=True).y_out

    ops = [symv, gemv_n, gemv_t, symv, through_panels, symv, gemv_n] * 3
    x0 = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=g)
    fast = _chain(ops, x0.clone(), sync=False)
    slow = _chain(ops, x0.clone(), sync=True)
    for i, (u, v) in enumerate(zip(fast, slow)):
        assert torch.equal(u, v), (i, float((u - v).abs().max()))
