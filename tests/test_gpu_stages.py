"""The reference's stage entry points (kernels.py:65-97 KernelRequest,
127-146 run_scal, 209-236 run_gemv_n / run_gemv_t, 287-313
run_symv_offdiag, 362-392 run_diag_block) on the B200 kernels, against
the oracle's restatement of the same stages (oracle/blocked.py) and the
reference's composition gemv = scal + accumulate, symv_hemv = diag +
offdiag (kernels.py:429-440, 471-486)."""

import numpy as np
import pytest
import torch

import paper_1410_1726_b200 as kb
from oracle import blocked, naive

pytestmark = pytest.mark.gpu


def dev_view(rng, m, n, tag, ld=None):
    ld = ld or -(-m // 32) * 32
    host = np.zeros(ld * n, dtype=naive.DTYPES[tag])
    win = naive.window(host, ld, m, n)
    win[:, :] = naive.fill(rng, (m, n), tag)
    return kb.MatrixView(torch.from_numpy(host).cuda(), m, n, ld, kb.precision(tag)), np.array(win)


def close(got, want, tag, scale):
    got = got.cpu().numpy() if isinstance(got, torch.Tensor) else np.asarray(got)
    assert got.dtype == want.dtype
    err = naive.max_abs_error(got, want)
    assert err <= 50 * naive.EPS[tag] * max(scale, 1.0), (err, scale)


@pytest.mark.parametrize("tag", "sdcz")
def test_run_scal(tag):
    rng = np.random.default_rng(1)
    p = kb.precision(tag)
    y = naive.fill(rng, 1000, tag)
    got = kb.run_scal(y, 2.5, p).y_out
    close(got, blocked.scal(y, 2.5, p.dtype), tag, float(np.max(np.abs(y))) * 2.5)
    ynan = y.copy()
    ynan[::7] = np.nan
    rep = kb.run_scal(ynan, 0.0, p)  # writes zeros without reading y (kernels.py:136-137)
    assert np.array_equal(rep.y_out, np.zeros_like(y)) and rep.flops == p.flops_per_mul * 1000
    yd = torch.from_numpy(y).cuda()
    assert isinstance(kb.run_scal(yd, -1.0, p).y_out, torch.Tensor)


@pytest.mark.parametrize("tag", "sdcz")
@pytest.mark.parametrize("op", ["n", "t", "c"])
def test_run_gemv_stages(tag, op):
    rng = np.random.default_rng(2)
    for m, n in [(300, 517), (1025, 64), (33, 2000)]:
        v, a = dev_view(rng, m, n, tag)
        xl, yl = (n, m) if op == "n" else (m, n)
        x, y = naive.fill(rng, xl, tag), naive.fill(rng, yl, tag)
        cfg = kb.KernelConfig(64, 4)
        if op == "n":
            rep = kb.run_gemv_n(kb.KernelRequest(kb.Op.GEMV_N, v, x, y, 0.75, 0.0, cfg))
            acc = blocked.gemv_accumulate(a, x, 0.75, 64, 1, False, False)
        else:
            rep = kb.run_gemv_t(kb.KernelRequest(kb.Op.GEMV_T, v, x, y, 0.75, 0.0, cfg), conjugate=op == "c")
            acc = blocked.gemv_accumulate(a, x, 0.75, 64, 1, True, op == "c" and tag in "cz")
        want = (y + acc).astype(naive.DTYPES[tag])
        dense = np.abs(a) if op == "n" else np.abs(a).T
        close(rep.y_out, want, tag, 0.75 * float(np.max(dense.sum(axis=1))) * float(np.max(np.abs(x)))
              + float(np.max(np.abs(y))))
        o, i = yl, xl
        p = kb.precision(tag)
        assert rep.flops == p.flops_per_mul * (o * i + o) + p.flops_per_add * (o * i)
    with pytest.raises(ValueError, match="expected GEMV_N request"):
        kb.run_gemv_n(kb.KernelRequest(kb.Op.GEMV_T, v, np.zeros(m), np.zeros(n), 1.0, 0.0, cfg))


@pytest.mark.parametrize("tag", "sdcz")
@pytest.mark.parametrize("uplo", "lu")
def test_symv_stages_compose_to_symv_hemv(tag, uplo):
    """run_diag_block (beta fused) then run_symv_offdiag on its output is
    the reference's symv_hemv (kernels.py:471-486) and matches the oracle
    stage by stage."""
    rng = np.random.default_rng(3)
    herm = tag in "cz"
    op = {("l", True): kb.Op.HEMV_LOWER, ("u", True): kb.Op.HEMV_UPPER,
          ("l", False): kb.Op.SYMV_LOWER, ("u", False): kb.Op.SYMV_UPPER}[(uplo, herm)]
    for d, nb in [(700, 64), (1000, 32), (257, 128)]:
        v, a = dev_view(rng, d, d, tag)
        hv = kb.HermitianView(v, uplo)
        x, y = naive.fill(rng, d, tag), naive.fill(rng, d, tag)
        cfg = kb.KernelConfig(nb, 2)
        diag = kb.run_diag_block(kb.KernelRequest(op, hv, x, y, 1.25, -0.5, cfg))
        dt = np.dtype(naive.DTYPES[tag])
        want_diag = (dt.type(-0.5) * y + blocked.diag_accumulate(a, uplo, x, 1.25, nb, herm)).astype(dt)
        full = np.abs(naive.dense_from_triangle(a, uplo, herm))
        scale = 1.25 * float(np.max(full.sum(axis=1))) * float(np.max(np.abs(x))) + 0.5 * float(np.max(np.abs(y)))
        close(diag.y_out, want_diag, tag, scale)
        off = kb.run_symv_offdiag(kb.KernelRequest(op, hv, x, diag.y_out, 1.25, -0.5, cfg))
        want_off = (diag.y_out + blocked.symv_offdiag_accumulate(a, uplo, x, 1.25, nb, 1, herm)).astype(dt)
        close(off.y_out, want_off, tag, scale)
        want = naive.naive_symv_hemv(1.25, a, uplo, x, -0.5, y, herm)
        close(off.y_out, want, tag, scale)
        t = -(-d // nb)
        diag_elems = (t - 1) * nb * nb + (d - (t - 1) * nb) ** 2
        p = kb.precision(tag)
        assert off.flops == (p.flops_per_mul + p.flops_per_add) * (d * d - diag_elems)
    with pytest.raises(ValueError, match="expected a symmetric/hermitian request"):
        kb.run_diag_block(kb.KernelRequest(kb.Op.GEMV_N, v, x, y, 1.0, 0.0, cfg))
