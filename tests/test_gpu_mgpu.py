"""mgpu API on the GPU (test_multidevice.py model).  Logical GPUs map onto
the physical devices present (all onto cuda:0 on a 1-GPU box)."""

import numpy as np
import pytest
import torch

import paper_1410_1726_b200 as kb
from oracle import blocked, naive

pytestmark = pytest.mark.gpu


def dev_matrix(rng, m, n, tag):
    ld = -(-m // 32) * 32
    host = np.zeros(ld * n, dtype=naive.DTYPES[tag])
    win = naive.window(host, ld, m, n)
    win[:, :] = naive.fill(rng, (m, n), tag)
    return kb.MatrixView(torch.from_numpy(host).cuda(), m, n, ld, kb.precision(tag)), np.array(win)


@pytest.mark.parametrize("devices", range(1, 9))
def test_distribute_gather_round_trip(devices):
    rng = np.random.default_rng(60 + devices)
    m, n = int(rng.integers(30, 200)), int(rng.integers(30, 200))
    v, a = dev_matrix(rng, m, n, "z")
    dist = kb.distribute(v, 32, devices)
    back = kb.gather(dist)
    assert torch.equal(back.array(), v.array())
    for g in range(devices):
        if dist.local_views[g] is None:
            assert not kb.owned_block_cols(n, 32, devices, g)


@pytest.mark.parametrize("devices", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("trans", "ntc")
def test_gemv_mgpu_matches_single(devices, trans):
    rng = np.random.default_rng(70)
    tag = "z" if trans == "c" else "d"
    for d in (64, 100, 256, 1000):
        v, a = dev_matrix(rng, d, d, tag)
        x, y = naive.fill(rng, d, tag), naive.fill(rng, d, tag)
        merged, per = kb.gemv_mgpu(trans, 1.2, kb.distribute(v, 32, devices), x, -0.5, y)
        single = kb.gemv(trans, 1.2, v, x, -0.5, y).y_out
        bound = naive.tolerance_bound(np.abs(a), x, tag) + 50 * naive.EPS[tag] * (np.max(np.abs(y)) + 1)
        assert naive.max_abs_error(merged.y_out, single) <= bound
        assert len(per) == devices
        assert merged.flops == sum(r.flops for r in per)


@pytest.mark.parametrize("devices", [1, 2, 4, 8])
@pytest.mark.parametrize("tag,uplo", [("d", "l"), ("d", "u"), ("c", "l"), ("z", "u"), ("s", "u")])
def test_symv_hemv_mgpu_matches_oracle(devices, tag, uplo):
    rng = np.random.default_rng(80)
    for d, nb in ((64, 32), (100, 32), (512, 64), (1500, 128)):
        v, a = dev_matrix(rng, d, d, tag)
        x, y = naive.fill(rng, d, tag), naive.fill(rng, d, tag)
        merged, per = kb.symv_hemv_mgpu(uplo, 0.9, kb.distribute(v, nb, devices), x, 0.7, y, kb.KernelConfig(nb, 2))
        want = naive.naive_symv_hemv(0.9, a, uplo, x, 0.7, y)
        sim = blocked.symv_hemv_mgpu(uplo, 0.9, a, x, 0.7, y, devices, nb)
        dense = np.abs(naive.dense_from_triangle(a, uplo, tag in "cz"))
        bound = naive.run_bound(tag, 0.9, dense, x, 0.7, y)
        assert naive.max_abs_error(merged.y_out, want) <= bound
        assert naive.max_abs_error(merged.y_out, sim) <= 2 * bound
        assert len(per) == devices


def test_transposed_segments_bit_identical_g1_g4():
    """test_multidevice.py:114-124: disjoint T segments, G=1 == G=4 bit-for-bit."""
    rng = np.random.default_rng(73)
    v, _ = dev_matrix(rng, 96, 96, "d")
    x = naive.fill(rng, 96, "d")
    y = np.zeros(96)
    one, _ = kb.gemv_mgpu("t", 1.0, kb.distribute(v, 32, 1), x, 0.0, y)
    four, _ = kb.gemv_mgpu("t", 1.0, kb.distribute(v, 32, 4), x, 0.0, y)
    assert np.array_equal(one.y_out, four.y_out)


def test_deterministic_reduction():
    rng = np.random.default_rng(72)
    v, _ = dev_matrix(rng, 1500, 1500, "s")
    x, y = naive.fill(rng, 1500, "s"), naive.fill(rng, 1500, "s")
    dist = kb.distribute(v, 32, 3)
    r1, _ = kb.gemv_mgpu("n", 1.0, dist, x, 0.3, y)
    r2, _ = kb.gemv_mgpu("n", 1.0, dist, x, 0.3, y)
    assert np.array_equal(r1.y_out, r2.y_out)


def test_symv_mgpu_validation():
    rng = np.random.default_rng(81)
    v, _ = dev_matrix(rng, 128, 128, "d")
    with pytest.raises(ValueError, match="block width"):
        kb.symv_hemv_mgpu("l", 1.0, kb.distribute(v, 64, 2), np.zeros(128), 0.0, np.zeros(128), kb.KernelConfig(32, 2))
    r, _ = dev_matrix(rng, 96, 64, "d")
    with pytest.raises(ValueError, match="square"):
        kb.symv_hemv_mgpu("l", 1.0, kb.distribute(r, 32, 2), np.zeros(64), 0.0, np.zeros(64), kb.KernelConfig(32, 2))


class TestCommandQueue:
    def test_results_unavailable_before_sync(self):
        rng = np.random.default_rng(90)
        v, a = dev_matrix(rng, 64, 64, "d")
        x, y = naive.fill(rng, 64, "d"), naive.fill(rng, 64, "d")
        q = kb.CommandQueue("stream-0")
        h = kb.gemv_mgpu_async("n", 1.0, kb.distribute(v, 32, 2), x, 0.0, y, kb.KernelConfig(32, 2), q)
        with pytest.raises(RuntimeError):
            h.result()
        q.synchronize()
        merged, per = h.result()
        assert np.allclose(merged.y_out, naive.naive_gemv("n", 1.0, a, x, 0.0, y))

    def test_in_order_execution(self):
        order = []
        q = kb.CommandQueue()
        q.submit(lambda: order.append("first"))
        q.submit(lambda: order.append("second"))
        q.synchronize()
        assert order == ["first", "second"]

    def test_symv_async(self):
        rng = np.random.default_rng(91)
        v, a = dev_matrix(rng, 96, 96, "d")
        x, y = naive.fill(rng, 96, "d"), naive.fill(rng, 96, "d")
        q = kb.CommandQueue()
        h = kb.symv_hemv_mgpu_async("l", 1.0, kb.distribute(v, 32, 3), x, 1.0, y, kb.KernelConfig(32, 2), q)
        q.synchronize()
        merged, _ = h.result()
        assert np.allclose(merged.y_out, naive.naive_symv_hemv(1.0, a, "l", x, 1.0, y))


class TestQueuedSingleGpu:
    """gemv_async / symv_hemv_async: the reference's queue contract on
    single-GPU calls.  numpy x and y are not waited for per call, so several
    calls are in flight with distinct results until synchronize()."""

    @pytest.mark.parametrize("tag", "dz")
    def test_numpy_calls_pipelined(self, tag):
        rng = np.random.default_rng(92)
        n = 1500
        v, a = dev_matrix(rng, n, n, tag)
        q = kb.CommandQueue()
        xs = [naive.fill(rng, n, tag) for _ in range(12)]
        y = naive.fill(rng, n, tag)
        hs = [kb.gemv_async("n", 1.0, v, x, 0.0, y, queue=q) for x in xs]
        hs += [kb.symv_hemv_async("l", 0.5, kb.HermitianView(v, "l"), x, -1.0, y, queue=q) for x in xs[:4]]
        with pytest.raises(RuntimeError):
            hs[0].result()
        q.synchronize()
        for x, h in zip(xs, hs[:12]):
            want = naive.naive_gemv("n", 1.0, a, x, 0.0, y)
            assert naive.max_abs_error(h.result().y_out, want) <= naive.run_bound(tag, 1.0, np.abs(a), x, 0.0, y)
        dense = np.abs(naive.dense_from_triangle(a, "l", tag in "cz"))
        for x, h in zip(xs[:4], hs[12:]):
            want = naive.naive_symv_hemv(0.5, a, "l", x, -1.0, y)
            assert naive.max_abs_error(h.result().y_out, want) <= naive.run_bound(tag, 0.5, dense, x, -1.0, y)
        # results are distinct buffers
        assert len({id(h.result().y_out) for h in hs}) == len(hs)

    def test_device_tensors_on_queue_stream(self):
        rng = np.random.default_rng(93)
        v, a = dev_matrix(rng, 640, 512, "s")
        x = torch.from_numpy(naive.fill(rng, 512, "s")).cuda()
        q = kb.CommandQueue()
        h = kb.gemv_async("n", 2.0, v, x, 0.0, torch.zeros(640, device="cuda"), queue=q)
        q.synchronize()
        want = naive.naive_gemv("n", 2.0, a, x.cpu().numpy(), 0.0, np.zeros(640, np.float32))
        got = h.result().y_out.cpu().numpy()
        assert naive.max_abs_error(got, want) <= naive.run_bound("s", 2.0, np.abs(a), x.cpu().numpy(), 0.0,
                                                                  np.zeros(640))


class TestFullSizeConfig5:
    """BASELINE configs[4] at its full size, N = 100000, where no host oracle
    fits: DSYMV lower over 2 logical GPUs (both on device 0), panels
    generated on the device.  Size-independent properties: the bilinear
    symmetry x^T (A y) = y^T (A x) of a symmetric operator, linearity in x,
    and agreement of G = 2 with the rank-order sum of the two per-GPU
    partials computed separately."""

    def test_dsymv_mgpu_100k_properties(self):
        free, _ = torch.cuda.mem_get_info()
        n, nb, G = 100000, 128, 2
        ld = kb.multidevice.local_ld(n)
        need = sum(kb.local_col_count(n, nb, G, g) for g in range(G)) * ld * 8
        if free < need + (8 << 30):
            pytest.skip(f"needs {need / 2**30:.0f} GiB of HBM")
        dev = torch.device("cuda", 0)
        gen = torch.Generator(device=dev).manual_seed(11)
        locals_ = []
        for g in range(G):
            lc = kb.local_col_count(n, nb, G, g)
            buf = torch.empty(lc * ld, dtype=torch.float64, device=dev)
            buf.uniform_(-1, 1, generator=gen)
            locals_.append(kb.MatrixView(buf, n, lc, ld, kb.precision("d")))
        dist = kb.DistributedMatrix(n, n, nb, G, kb.precision("d"), locals_, [dev] * G)
        cfg = kb.KernelConfig(nb, 2)
        x = torch.empty(n, dtype=torch.float64, device=dev).uniform_(-1, 1, generator=gen)
        y = torch.empty(n, dtype=torch.float64, device=dev).uniform_(-1, 1, generator=gen)
        zero = torch.zeros(n, dtype=torch.float64, device=dev)
        ax = kb.symv_hemv_mgpu("l", 1.0, dist, x, 0.0, zero, cfg)[0].y_out
        ay = kb.symv_hemv_mgpu("l", 1.0, dist, y, 0.0, zero, cfg)[0].y_out
        axy = kb.symv_hemv_mgpu("l", 1.0, dist, x + 2.0 * y, 0.0, zero, cfg)[0].y_out
        # |A|_inf <= n for U(-1,1) entries; error bounds c * n * eps * |A| |x|
        eps = np.finfo(np.float64).eps
        scale = float(n) * float(x.abs().max()) * float(y.abs().max())
        lhs, rhs = float(torch.dot(x, ay)), float(torch.dot(y, ax))
        assert abs(lhs - rhs) <= 50 * n * eps * scale
        lin = (axy - (ax + 2.0 * ay)).abs().max().item()
        assert lin <= 50 * n * eps * float(n) * 3.0
        # G = 2 equals the rank-order sum of the two partials
        parts = []
        for g in range(G):
            out = torch.empty(n, dtype=torch.float64, device=dev)
            kb.partial_mv(kb.precision("d"), "s", "l", n, n, 1.0, locals_[g], x, out, G, g, nb)
            parts.append(out)
        assert torch.equal(parts[0] + parts[1], ax)
        # beta path: y_out = beta*y + A x
        r = kb.symv_hemv_mgpu("l", 1.0, dist, x, -0.5, y, cfg)[0].y_out
        assert (r - (ax - 0.5 * y)).abs().max().item() <= 4 * eps * float((ax.abs() + y.abs()).max())


# property form: random shapes, block widths, GPU counts, reduce modes,
# scalars and vector kinds against the single-GPU API
import os  # noqa: E402

from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@settings(max_examples=int(os.environ.get("KB_HYP_EXAMPLES", 60)), deadline=None,
          derandomize=not os.environ.get("KB_HYP_RANDOM"),
          suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])
@given(tag=st.sampled_from("sdcz"), kind=st.sampled_from(["gemv", "symv"]), m=st.integers(1, 1500),
       n=st.integers(1, 1500), nb_pow=st.integers(4, 8), devices=st.integers(1, 8),
       op=st.sampled_from("ntclu"), reduce=st.sampled_from(["ordered", "nccl"]),
       beta=st.sampled_from([0.0, 1.0, -0.5]), numpy_vecs=st.booleans(), seed=st.integers(0, 2 ** 16))
def test_mgpu_property(tag, kind, m, n, nb_pow, devices, op, reduce, beta, numpy_vecs, seed):
    rng = np.random.default_rng(seed)
    nb = 1 << nb_pow
    if kind == "symv":
        n = m
        op = op if op in "lu" else "l"
    else:
        op = op if op in "ntc" else "n"
    v, a = dev_matrix(rng, m, n, tag)
    xl, yl = (n, m) if (kind == "gemv" and op == "n") else ((m, n) if kind == "gemv" else (m, m))
    x, y = naive.fill(rng, xl, tag), naive.fill(rng, yl, tag)
    if not numpy_vecs:
        x, y = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    dist_mat = kb.distribute(v, nb, devices)
    if kind == "symv":
        herm = tag in "cz"
        merged, per = kb.symv_hemv_mgpu(op, 0.8, dist_mat, x, beta, y, kb.KernelConfig(nb, 2), hermitian=herm,
                                        reduce=reduce)
        single = kb.symv_hemv(op, 0.8, kb.HermitianView(v, op), x, beta, y, hermitian=herm).y_out
        dense = np.abs(naive.dense_from_triangle(a, op, herm))
    else:
        merged, per = kb.gemv_mgpu(op, 0.8, dist_mat, x, beta, y, reduce=reduce)
        single = kb.gemv(op, 0.8, v, x, beta, y).y_out
        dense = np.abs(a) if op == "n" else np.abs(a).T
    got = merged.y_out.cpu().numpy() if isinstance(merged.y_out, torch.Tensor) else merged.y_out
    want = single.cpu().numpy() if isinstance(single, torch.Tensor) else single
    assert type(merged.y_out) is type(single)
    xh = x.cpu().numpy() if isinstance(x, torch.Tensor) else x
    yh = y.cpu().numpy() if isinstance(y, torch.Tensor) else y
    bound = 2 * naive.run_bound(tag, 0.8, dense, xh, beta, yh)
    assert naive.max_abs_error(got, want) <= bound
    assert len(per) == devices
