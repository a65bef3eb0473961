"""Numpy-vector calls (the reference's numpy-in / numpy-out call shape,
kernels.py:402-486) through kblas_mv_hostvec and its CPython binding.

Page-locked x / y are staged by the copy-in grid and the main kernel is
launched as its programmatic dependent (A prefetched before
griddepcontrol.wait); pageable ones go through the copy engine.  Both must
give exactly the result of the device-tensor call (same plan, same
kernels), for every op and precision, misaligned page-locked views
(4-byte copy path) included, and back-to-back queued calls must not see
each other's staging."""

import os

import numpy as np
import pytest
import torch

import paper_1410_1726_b200 as kb
from oracle import naive

pytestmark = pytest.mark.gpu

DT = {"s": torch.float32, "d": torch.float64, "c": torch.complex64, "z": torch.complex128}


def pinned(a, shift=0):
    """Copy of a in page-locked memory, starting `shift` elements into the
    allocation (shift > 0: not 16-byte aligned for 8/16-byte elements).
    The numpy view keeps the torch allocation alive."""
    a = np.asarray(a)
    t = torch.empty(a.size + shift, dtype=DT[_tag(a)], pin_memory=True)
    h = t.numpy()[shift:]
    h[:] = a
    return h


def _tag(a):
    return {np.float32: "s", np.float64: "d", np.complex64: "c", np.complex128: "z"}[np.dtype(a.dtype).type]


def dev_view(rng, m, n, tag, ld=None, host=True):
    """(MatrixView in HBM, host copy of the m x n window or None).  Large
    operands are filled on the device (host=False): the tests compare the
    host-vector call with the device-tensor call bit for bit."""
    ld = ld or -(-m // 32) * 32
    if not host:
        g = torch.Generator(device="cuda").manual_seed(int(rng.integers(1 << 31)))
        t = torch.empty(ld * n, dtype=DT[tag], device="cuda")
        (torch.view_as_real(t) if tag in "cz" else t).uniform_(-1, 1, generator=g)
        return kb.MatrixView(t, m, n, ld, kb.precision(tag)), None
    buf = np.zeros(ld * n, dtype=naive.DTYPES[tag])
    win = naive.window(buf, ld, m, n)
    win[:, :] = naive.fill(rng, (m, n), tag)
    return kb.MatrixView(torch.from_numpy(buf).cuda(), m, n, ld, kb.precision(tag)), np.array(win)


def same(got, want):
    got = np.asarray(got)
    want = want.cpu().numpy() if isinstance(want, torch.Tensor) else np.asarray(want)
    assert got.dtype == want.dtype and got.shape == want.shape
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, (f"{bad.size} of {got.size} differ, first {bad[:5].tolist()}, last {bad[-5:].tolist()}, "
                           f"max {float(np.max(np.abs(got - want)))}")


@pytest.mark.parametrize("tag", "sdcz")
@pytest.mark.parametrize("trans", "ntc")
@pytest.mark.parametrize("kind", ["pinned", "pinned_shifted", "pageable"])
def test_gemv_hostvec_equals_device_path(tag, trans, kind):
    rng = np.random.default_rng(101)
    for m, n, beta in [(4096, 4096, 0.0), (1000, 37, 0.5), (37, 1000, 0.0), (2049, 1537, -1.25)]:
        v, a = dev_view(rng, m, n, tag, host=m * n < 4_000_000)
        xl, yl = (n, m) if trans == "n" else (m, n)
        x, y = naive.fill(rng, xl, tag), naive.fill(rng, yl, tag)
        if kind == "pinned":
            hx, hy = pinned(x), pinned(y)
        elif kind == "pinned_shifted":
            hx, hy = pinned(x, 1), pinned(y, 1)
        else:
            hx, hy = x.copy(), y.copy()
        got = kb.gemv(trans, 0.7, v, hx, beta, hy).y_out
        want = kb.gemv(trans, 0.7, v, torch.from_numpy(x).cuda(), beta, torch.from_numpy(y).cuda()).y_out
        same(got, want)
        if a is not None:  # and within the reference bound of the oracle
            ref = naive.naive_gemv(trans, 0.7, a, x, beta, y)
            dense = np.abs(a) if trans == "n" else np.abs(a).T
            assert naive.max_abs_error(got, ref) <= naive.run_bound(tag, 0.7, dense, x, beta, y)
        # inputs not mutated
        assert np.array_equal(hx, x) and np.array_equal(hy, y)


@pytest.mark.parametrize("tag", "sdcz")
@pytest.mark.parametrize("uplo", "lu")
@pytest.mark.parametrize("kind", ["pinned", "pinned_shifted", "pageable"])
def test_symv_hemv_hostvec_equals_device_path(tag, uplo, kind):
    rng = np.random.default_rng(102)
    herm = tag in "cz"
    for d, beta in [(4096, 0.0), (1001, 0.5), (12288, 0.0)]:
        v, a = dev_view(rng, d, d, tag, host=False)
        hv = kb.HermitianView(v, uplo)
        x, y = naive.fill(rng, d, tag), naive.fill(rng, d, tag)
        if kind == "pinned":
            hx, hy = pinned(x), pinned(y)
        elif kind == "pinned_shifted":
            hx, hy = pinned(x, 1), pinned(y, 1)
        else:
            hx, hy = x.copy(), y.copy()
        got = kb.symv_hemv(uplo, 1.5, hv, hx, beta, hy, hermitian=herm).y_out
        want = kb.symv_hemv(uplo, 1.5, hv, torch.from_numpy(x).cuda(), beta, torch.from_numpy(y).cuda(),
                            hermitian=herm).y_out
        same(got, want)


@pytest.mark.parametrize("tag", "sdcz")
@pytest.mark.parametrize("kind", ["pinned", "pageable"])
def test_offset_hostvec(tag, kind):
    """The offset entry points take the same host-vector path (with the
    offsets passed to kblas_mv_hostvec) and match the device-tensor call."""
    rng = np.random.default_rng(103)
    v, a = dev_view(rng, 2048, 2048, tag, host=False)
    conv = pinned if kind == "pinned" else (lambda z: z.copy())
    for (i, j) in [(7, 3), (13, 13), (16, 16)]:
        req = kb.OffsetRequest(v, i, j, 2048 - i, 2048 - j)
        for trans in "ntc":
            xl, yl = (req.sub_n, req.sub_m) if trans == "n" else (req.sub_m, req.sub_n)
            x, y = naive.fill(rng, xl, tag), naive.fill(rng, yl, tag)
            for beta in (0.0, 0.25):
                got = kb.gemv_offset(trans, 0.5, req, conv(x), beta, conv(y)).y_out
                want = kb.gemv_offset(trans, 0.5, req, torch.from_numpy(x).cuda(), beta,
                                      torch.from_numpy(y).cuda()).y_out
                same(got, want)
    for uplo in "lu":
        hv = kb.HermitianView(v, uplo)
        for off in (1, 13, 16):
            d = 2048 - off
            x, y = naive.fill(rng, d, tag), naive.fill(rng, d, tag)
            for beta in (0.0, 0.25):
                got = kb.symv_hemv_offset(uplo, 0.5, hv, off, d, conv(x), beta, conv(y)).y_out
                want = kb.symv_hemv_offset(uplo, 0.5, hv, off, d, torch.from_numpy(x).cuda(), beta,
                                           torch.from_numpy(y).cuda()).y_out
                same(got, want)


def test_offset_hostvec_errors():
    rng = np.random.default_rng(107)
    v, a = dev_view(rng, 64, 64, "d")
    req = kb.OffsetRequest(v, 1, 1, 63, 63)
    with pytest.raises(ValueError, match="expected x of length 63 and y of length 63"):
        kb.gemv_offset("n", 1.0, req, np.zeros(62), 0.0, np.zeros(63))
    with pytest.raises(ValueError, match="expected x and y of length 63"):
        kb.symv_hemv_offset("l", 1.0, kb.HermitianView(v, "l"), 1, 63, np.zeros(63), 0.0, np.zeros(64))


@pytest.mark.parametrize("op", ["gemv", "symv"])
def test_queued_pinned_calls_do_not_share_staging(op):
    """Many queued calls with different page-locked x: each result is its
    own (the staging buffer of call i+1 is written only after call i's
    kernels have finished with it)."""
    rng = np.random.default_rng(104)
    n = 4096
    v, a = dev_view(rng, n, n, "d", host=False)
    hv = kb.HermitianView(v, "l")
    q = kb.CommandQueue()
    xs = [pinned(naive.fill(rng, n, "d")) for _ in range(24)]
    y = np.zeros(n)
    hs = []
    for x in xs:
        if op == "gemv":
            hs.append(kb.gemv_async("n", 1.0, v, x, 0.0, y, queue=q))
        else:
            hs.append(kb.symv_hemv_async("l", 1.0, hv, x, 0.0, y, queue=q))
    with pytest.raises(RuntimeError, match="queue not synchronized yet"):
        hs[0].result()
    q.synchronize()
    for x, h in zip(xs, hs):
        xd = torch.from_numpy(np.array(x)).cuda()
        if op == "gemv":
            want = kb.gemv("n", 1.0, v, xd, 0.0, torch.zeros(n, dtype=torch.float64, device="cuda")).y_out
        else:
            want = kb.symv_hemv("l", 1.0, hv, xd, 0.0, torch.zeros(n, dtype=torch.float64, device="cuda")).y_out
        same(h.result().y_out, want)
        assert h.result().flops > 0  # the deferred report fills on access


@pytest.mark.parametrize("tag", "dz")
def test_queued_mixed_calls(tag):
    """A long queue mixing every form of the host-vector path on one stream
    (row-owning and split GEMV-N, GEMV-T/C, SYMV/HEMV with its epilogue,
    beta != 0 with y staged, alpha = 0 scal, a 100k-element x that takes
    several copy-in passes, shifted page-locked views): each copy-in grid
    starts while the previous call drains and writes the shared staging
    buffer only after it, so every result equals its device-tensor call."""
    rng = np.random.default_rng(106)
    dt = naive.DTYPES[tag]
    sq, _ = dev_view(rng, 2048, 2048, tag, host=False)
    tall, _ = dev_view(rng, 100000, 48, tag, host=False)
    wide, _ = dev_view(rng, 300, 6000, tag, host=False)
    hv = kb.HermitianView(sq, "l")
    herm = tag in "cz"
    calls = []
    for i in range(48):
        kind = ["gemv_sq", "symv", "gemv_t_tall", "gemv_n_wide", "scal", "gemv_c_sq"][i % 6]
        beta = 0.0 if i % 4 else -0.5
        shift = i % 3 == 2
        if kind == "gemv_sq":
            args = ("n", 0.75, sq, 2048, 2048)
        elif kind == "gemv_c_sq":
            args = ("c", 0.75, sq, 2048, 2048)
        elif kind == "gemv_t_tall":
            args = ("t", 1.25, tall, 100000, 48)
        elif kind == "gemv_n_wide":
            args = ("n", 1.25, wide, 6000, 300)
        elif kind == "scal":
            args = ("n", 0.0, sq, 2048, 2048)
        else:
            args = None
        if kind == "symv":
            x = pinned(naive.fill(rng, 2048, tag), 1 if shift else 0)
            y = pinned(naive.fill(rng, 2048, tag))
            calls.append((kind, x, y, beta, None))
        else:
            trans, alpha, view, xl, yl = args
            x = pinned(naive.fill(rng, xl, tag), 1 if shift else 0)
            y = pinned(naive.fill(rng, yl, tag))
            calls.append((kind, x, y, beta, (trans, alpha, view)))
    q = kb.CommandQueue()
    hs = []
    for kind, x, y, beta, g in calls:
        if kind == "symv":
            hs.append(kb.symv_hemv_async("l", 0.5, hv, x, beta, y, queue=q, hermitian=herm))
        else:
            trans, alpha, view = g
            hs.append(kb.gemv_async(trans, alpha, view, x, beta, y, queue=q))
    q.synchronize()
    for (kind, x, y, beta, g), h in zip(calls, hs):
        xd = torch.from_numpy(np.array(x, dtype=dt)).cuda()
        yd = torch.from_numpy(np.array(y, dtype=dt)).cuda()
        if kind == "symv":
            want = kb.symv_hemv("l", 0.5, hv, xd, beta, yd, hermitian=herm).y_out
        else:
            trans, alpha, view = g
            want = kb.gemv(trans, alpha, view, xd, beta, yd).y_out
        same(h.result().y_out, want)


def test_queue_orders_after_callers_stream():
    """A queued call sees work the caller enqueued on its own stream before
    submitting (kblas_stream_order), without a host wait."""
    rng = np.random.default_rng(105)
    n = 2048
    v, a = dev_view(rng, n, n, "d")
    q = kb.CommandQueue()
    x = pinned(naive.fill(rng, n, "d"))
    # a long kernel on the caller's stream that rewrites A just before the call
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        torch.cuda._sleep(20_000_000)
        v.data.mul_(2.0)
        h = kb.gemv_async("n", 1.0, v, x, 0.0, np.zeros(n), queue=q)
    q.synchronize()
    want = kb.gemv("n", 1.0, v, torch.from_numpy(np.array(x)).cuda(), 0.0,
                   torch.zeros(n, dtype=torch.float64, device="cuda")).y_out
    same(h.result().y_out, want)


def test_hostvec_report_counters():
    rng = np.random.default_rng(106)
    v, a = dev_view(rng, 512, 256, "z")
    x, y = naive.fill(rng, 256, "z"), naive.fill(rng, 512, "z")
    rep = kb.gemv("n", 1.0, v, pinned(x), 0.0, pinned(y))
    dev = kb.gemv("n", 1.0, v, torch.from_numpy(x).cuda(), 0.0, torch.from_numpy(y).cuda())
    for f in ("bytes_read", "bytes_written", "transactions", "matrix_transactions", "flops", "tb_count",
              "reduction_events", "scal_invocations", "plan"):
        assert getattr(rep, f) == getattr(dev, f), f


# property form: random shapes, views, scalars and vector memory kinds
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@settings(max_examples=int(os.environ.get("KB_HYP_EXAMPLES", 120)), deadline=None,
          derandomize=not os.environ.get("KB_HYP_RANDOM"),
          suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])
@given(tag=st.sampled_from("sdcz"), kind=st.sampled_from(["gemv", "symv"]), m=st.integers(1, 3000),
       n=st.integers(1, 3000), op=st.sampled_from("ntclu"), mem=st.sampled_from(["pinned", "shifted", "pageable"]),
       alpha=st.sampled_from([1.0, -0.5, 2.25]), beta=st.sampled_from([0.0, 1.0, -0.75]),
       queued=st.booleans(), off=st.sampled_from([0, 0, 1, 7, 13]), seed=st.integers(0, 2 ** 16))
def test_hostvec_property(tag, kind, m, n, op, mem, alpha, beta, queued, off, seed):
    """Any shape and op: the numpy-vector call (sync or queued; off > 0:
    the offset API on a parent `off` rows/columns larger) gives the
    device-tensor call's result bit for bit."""
    rng = np.random.default_rng(seed)
    if kind == "symv":
        n = m
        op = op if op in "lu" else "l"
    else:
        op = op if op in "ntc" else "n"
    if off:
        queued = False  # the offset API has no queued form
        pv, _ = dev_view(rng, m + off, n + off, tag, host=False)
        xl, yl = (m, m) if kind == "symv" else ((n, m) if op == "n" else (m, n))
        x, y = naive.fill(rng, xl, tag), naive.fill(rng, yl, tag)
        conv = {"pinned": pinned, "shifted": lambda a: pinned(a, 1), "pageable": lambda a: a.copy()}[mem]
        dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        if kind == "symv":
            hv = kb.HermitianView(pv, op)
            want = kb.symv_hemv_offset(op, alpha, hv, off, m, dx, beta, dy).y_out
            got = kb.symv_hemv_offset(op, alpha, hv, off, m, conv(x), beta, conv(y)).y_out
        else:
            req = kb.OffsetRequest(pv, off, off // 2, m, n)
            want = kb.gemv_offset(op, alpha, req, dx, beta, dy).y_out
            got = kb.gemv_offset(op, alpha, req, conv(x), beta, conv(y)).y_out
        same(got, want)
        return
    v, _ = dev_view(rng, m, n, tag, host=False)
    xl, yl = (m, m) if kind == "symv" else ((n, m) if op == "n" else (m, n))
    x, y = naive.fill(rng, xl, tag), naive.fill(rng, yl, tag)
    conv = {"pinned": pinned, "shifted": lambda a: pinned(a, 1), "pageable": lambda a: a.copy()}[mem]
    hx, hy = conv(x), conv(y)
    herm = tag in "cz"
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    if kind == "symv":
        hv = kb.HermitianView(v, op)
        want = kb.symv_hemv(op, alpha, hv, dx, beta, dy, hermitian=herm).y_out
        if queued:
            q = kb.CommandQueue()
            h = kb.symv_hemv_async(op, alpha, hv, hx, beta, hy, queue=q, hermitian=herm)
            q.synchronize()
            got = h.result().y_out
        else:
            got = kb.symv_hemv(op, alpha, hv, hx, beta, hy, hermitian=herm).y_out
    else:
        want = kb.gemv(op, alpha, v, dx, beta, dy).y_out
        if queued:
            q = kb.CommandQueue()
            h = kb.gemv_async(op, alpha, v, hx, beta, hy, queue=q)
            q.synchronize()
            got = h.result().y_out
        else:
            got = kb.gemv(op, alpha, v, hx, beta, hy).y_out
    same(got, want)


def test_threads_share_a_stream():
    """Four host threads issue numpy-vector calls on the same (default)
    stream at once: each call's acquire-and-launch sequence holds the
    per-(device, stream) lock, so the shared staging buffer and workspace
    are never interleaved, and every result is its own."""
    import threading

    rng = np.random.default_rng(108)
    n = 2048
    v, _ = dev_view(rng, n, n, "d", host=False)
    hv = kb.HermitianView(v, "l")
    xs = [naive.fill(rng, n, "d") for _ in range(4)]
    wants = []
    for x in xs:
        xd = torch.from_numpy(x).cuda()
        z = torch.zeros(n, dtype=torch.float64, device="cuda")
        wants.append((kb.gemv("n", 1.0, v, xd, 0.0, z).y_out.cpu().numpy(),
                      kb.symv_hemv("l", 1.0, hv, xd, 0.0, z).y_out.cpu().numpy()))
    errors = []

    def work(t):
        try:
            hx = pinned(xs[t], t % 2)
            for i in range(50):
                if i % 2:
                    got = kb.symv_hemv("l", 1.0, hv, hx, 0.0, np.zeros(n)).y_out
                    ok = np.array_equal(got, wants[t][1])
                else:
                    got = kb.gemv("n", 1.0, v, hx, 0.0, np.zeros(n)).y_out
                    ok = np.array_equal(got, wants[t][0])
                if not ok:
                    errors.append((t, i))
        except Exception as e:  # pragma: no cover - reported below
            errors.append((t, repr(e)))

    threads = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert errors == []
