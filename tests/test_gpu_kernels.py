"""GPU behaviour and parity tests modelled on the reference's own tests
(test_kernels.py, test_offset.py, test_acceptance.py c1/c5/c8), run
through the drop-in API and the C ABI against the CPU oracle."""

import ctypes

import numpy as np
import pytest
import torch

import paper_1410_1726_b200 as kb
from paper_1410_1726_b200 import _lib, tuner
from oracle import naive, streamed

pytestmark = pytest.mark.gpu

DT = {"s": torch.float32, "d": torch.float64, "c": torch.complex64, "z": torch.complex128}


def dev_matrix(rng, m, n, tag, ld=None, fill=naive.fill):
    """(MatrixView on the GPU, host 2-D copy) with leading dimension ld."""
    ld = ld or m
    host = np.zeros(ld * n, dtype=naive.DTYPES[tag])
    win = naive.window(host, ld, m, n)
    win[:, :] = fill(rng, (m, n), tag)
    v = kb.MatrixView(torch.from_numpy(host).cuda(), m, n, ld, kb.precision(tag))
    return v, np.array(win)


def dvec(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check(got, want, tag, alpha, dense_abs, x, beta, y, factor=1.0):
    got = got.cpu().numpy() if isinstance(got, torch.Tensor) else got
    bound = factor * naive.run_bound(tag, alpha, dense_abs, x, beta, y)
    err = naive.max_abs_error(got, want)
    assert err <= bound, (err, bound)


class TestGemv:
    @pytest.mark.parametrize("tag", "sdcz")
    @pytest.mark.parametrize("trans", "ntc")
    def test_matches_oracle_shapes(self, tag, trans):
        """test_kernels.py:42-55 shapes plus wave-edge and ragged sizes."""
        rng = np.random.default_rng(11)
        for m, n in [(1, 1), (7, 5), (32, 32), (65, 33), (100, 300), (1000, 37), (37, 1000), (2049, 1537)]:
            v, a = dev_matrix(rng, m, n, tag, ld=-(-m // 32) * 32)
            xl, yl = (n, m) if trans == "n" else (m, n)
            x, y = naive.fill(rng, xl, tag), naive.fill(rng, yl, tag)
            got = kb.gemv(trans, 0.7, v, dvec(x), -0.3, dvec(y)).y_out
            want = naive.naive_gemv(trans, 0.7, a, x, -0.3, y)
            dense = np.abs(a) if trans == "n" else np.abs(a).T
            check(got, want, tag, 0.7, dense, x, -0.3, y)

    @pytest.mark.parametrize("tag", "sdcz")
    def test_every_lead_and_unaligned_ld(self, tag):
        """Submatrix starts at every offset inside the 32-byte granule
        (realigned 256-bit path) and odd ld (one-element path)."""
        rng = np.random.default_rng(12)
        for ld in (515, 520):
            v, a = dev_matrix(rng, 500, 300, tag, ld=ld)
            for ro in range(0, 9):
                for trans in "nt":
                    sub = v.submatrix(ro, 3, 480 - ro, 290)
                    sa = a[ro:480, 3:293]
                    xl, yl = (290, 480 - ro) if trans == "n" else (480 - ro, 290)
                    x, y = naive.fill(rng, xl, tag), naive.fill(rng, yl, tag)
                    got = kb.gemv(trans, 1.3, sub, dvec(x), 0.5, dvec(y)).y_out
                    want = naive.naive_gemv(trans, 1.3, sa, x, 0.5, y)
                    dense = np.abs(sa) if trans == "n" else np.abs(sa).T
                    check(got, want, tag, 1.3, dense, x, 0.5, y)

    def test_deterministic(self):
        """Bit-identical repeated calls (test_kernels.py:57-65): no atomics."""
        rng = np.random.default_rng(3)
        for tag in "sz":
            v, _ = dev_matrix(rng, 3000, 2000, tag)
            for trans in "nt":
                xl, yl = (2000, 3000) if trans == "n" else (3000, 2000)
                x, y = dvec(naive.fill(rng, xl, tag)), dvec(naive.fill(rng, yl, tag))
                r1 = kb.gemv(trans, 1.3, v, x, 0.4, y).y_out
                r2 = kb.gemv(trans, 1.3, v, x, 0.4, y).y_out
                assert torch.equal(r1, r2)

    def test_beta_zero_kills_nan(self):
        rng = np.random.default_rng(6)
        v, a = dev_matrix(rng, 64, 64, "d")
        x = naive.fill(rng, 64, "d")
        for trans in "nt":
            got = kb.gemv(trans, 1.0, v, dvec(x), 0.0, torch.full((64,), float("nan"), device="cuda")).y_out
            assert torch.isfinite(got).all()
            check(got, naive.naive_gemv(trans, 1.0, a, x, 0.0, np.zeros(64)), "d", 1.0, np.abs(a), x, 0.0,
                  np.zeros(64))

    def test_quick_return_and_alpha_zero(self):
        rng = np.random.default_rng(7)
        v, a = dev_matrix(rng, 32, 32, "d")
        x, y = naive.fill(rng, 32, "d"), naive.fill(rng, 32, "d")
        n0 = _lib.launch_count()
        rep = kb.gemv("n", 0.0, v, dvec(x), 1.0, dvec(y))
        assert np.array_equal(rep.y_out.cpu().numpy(), y)
        assert rep.transactions == 0 and rep.tb_count == 0 and rep.flops == 0
        assert _lib.launch_count() == n0
        # alpha == 0: beta * y only, A never read (poison it)
        v.data.fill_(float("nan"))
        rep = kb.gemv("n", 0.0, v, dvec(x), 0.5, dvec(y))
        assert np.allclose(rep.y_out.cpu().numpy(), 0.5 * y)
        assert rep.matrix_transactions == 0 and rep.scal_invocations == 1

    def test_conjugate_on_real_is_transpose_bit_exact(self):
        rng = np.random.default_rng(13)
        v, _ = dev_matrix(rng, 40, 30, "d")
        x, y = dvec(naive.fill(rng, 40, "d")), dvec(naive.fill(rng, 30, "d"))
        assert torch.equal(kb.gemv("c", 1.0, v, x, 0.0, y).y_out, kb.gemv("t", 1.0, v, x, 0.0, y).y_out)

    def test_inputs_not_mutated_and_types(self):
        rng = np.random.default_rng(14)
        v, a = dev_matrix(rng, 50, 40, "z")
        x, y = naive.fill(rng, 40, "z"), naive.fill(rng, 50, "z")
        xt, yt = dvec(x), dvec(y)
        before = v.data.clone()
        rep = kb.gemv("n", 1 + 2j, v, xt, 0.5 - 1j, yt)
        assert torch.equal(v.data, before) and np.array_equal(yt.cpu().numpy(), y)
        assert isinstance(rep.y_out, torch.Tensor) and rep.y_out.dtype == torch.complex128
        rep2 = kb.gemv("n", 1 + 2j, v, x, 0.5 - 1j, y)
        assert isinstance(rep2.y_out, np.ndarray)
        assert np.array_equal(rep2.y_out, rep.y_out.cpu().numpy())

    def test_inplace(self):
        rng = np.random.default_rng(15)
        v, a = dev_matrix(rng, 300, 200, "d")
        x, y = naive.fill(rng, 200, "d"), naive.fill(rng, 300, "d")
        yt = dvec(y)
        rep = kb.gemv("n", 2.0, v, dvec(x), 1.5, yt, inplace=True)
        assert rep.y_out.data_ptr() == yt.data_ptr()
        check(yt, naive.naive_gemv("n", 2.0, a, x, 1.5, y), "d", 2.0, np.abs(a), x, 1.5, y)

    def test_errors(self):
        rng = np.random.default_rng(16)
        v, _ = dev_matrix(rng, 8, 8, "d")
        with pytest.raises(ValueError):
            kb.gemv("q", 1.0, v, np.zeros(8), 0.0, np.zeros(8))
        with pytest.raises(ValueError):
            kb.gemv("n", 1.0, v, np.zeros(7), 0.0, np.zeros(8))


class TestSymv:
    @pytest.mark.parametrize("tag", "sdcz")
    @pytest.mark.parametrize("uplo", "lu")
    def test_matches_oracle_sizes(self, tag, uplo):
        """test_kernels.py:166-179 sizes plus tile-edge sizes."""
        rng = np.random.default_rng(21)
        for d in (1, 5, 32, 33, 100, 127, 128, 129, 257, 1000, 2047):
            for herm in ([True, False] if tag in "cz" else [False]):
                v, a = dev_matrix(rng, d, d, tag, ld=-(-d // 32) * 32)
                x, y = naive.fill(rng, d, tag), naive.fill(rng, d, tag)
                hv = kb.HermitianView(v, uplo)
                got = kb.symv_hemv(uplo, 1.1, hv, dvec(x), -0.2, dvec(y), hermitian=herm).y_out
                want = naive.naive_symv_hemv(1.1, a, uplo, x, -0.2, y, hermitian=herm)
                dense = np.abs(naive.dense_from_triangle(a, uplo, herm))
                check(got, want, tag, 1.1, dense, x, -0.2, y)

    @pytest.mark.parametrize("tag", "sdcz")
    @pytest.mark.parametrize("uplo", "lu")
    def test_unreferenced_triangle_poisoned(self, tag, uplo):
        """The other triangle holds NaN: result must be finite and correct
        (the executable form of the reference's triangle guard,
        core.py:155-188, test_kernels.py:213-221)."""
        rng = np.random.default_rng(25)
        for d, ro in ((300, 0), (517, 3), (1024, 1)):
            ld = d + 8
            host = np.full(ld * d, np.nan, dtype=naive.DTYPES[tag])
            win = naive.window(host, ld, d, d)
            vals = naive.fill(rng, (d - ro, d - ro), tag)
            tri = np.tril(vals) if uplo == "l" else np.triu(vals)
            mask = np.tril(np.ones((d - ro,) * 2, bool)) if uplo == "l" else np.triu(np.ones((d - ro,) * 2, bool))
            sub = win[ro:, ro:]
            sub[mask] = tri[mask]
            v = kb.MatrixView(torch.from_numpy(host).cuda(), d, d, ld, kb.precision(tag)).submatrix(
                ro, ro, d - ro, d - ro)
            x, y = naive.fill(rng, d - ro, tag), naive.fill(rng, d - ro, tag)
            got = kb.symv_hemv(uplo, 0.9, kb.HermitianView(v, uplo), dvec(x), 0.0, dvec(y)).y_out
            assert torch.isfinite(got).all()
            herm = tag in "cz"
            want = naive.naive_symv_hemv(0.9, tri, uplo, x, 0.0, y, hermitian=herm)
            check(got, want, tag, 0.9, np.abs(naive.dense_from_triangle(tri, uplo, herm)), x, 0.0, y)

    def test_hemv_ignores_imaginary_diagonal(self):
        rng = np.random.default_rng(26)
        d = 200
        v, a = dev_matrix(rng, d, d, "c")
        idx = np.arange(d)
        a[idx, idx] = a[idx, idx].real + 5j
        v.array().copy_(torch.from_numpy(a).cuda())
        x, y = naive.fill(rng, d, "c"), naive.fill(rng, d, "c")
        got = kb.hemv("l", 1.0, kb.HermitianView(v, "l"), dvec(x), 0.0, dvec(y)).y_out
        want = naive.naive_symv_hemv(1.0, a, "l", x, 0.0, y, hermitian=True)
        check(got, want, "c", 1.0, np.abs(naive.dense_from_triangle(a, "l", True)), x, 0.0, y)

    def test_deterministic_and_no_scal(self):
        rng = np.random.default_rng(22)
        v, _ = dev_matrix(rng, 3000, 3000, "d")
        hv = kb.HermitianView(v, "l")
        x, y = dvec(naive.fill(rng, 3000, "d")), dvec(naive.fill(rng, 3000, "d"))
        r1 = kb.symv_hemv("l", 1.0, hv, x, 3.0, y)
        r2 = kb.symv_hemv("l", 1.0, hv, x, 3.0, y)
        assert torch.equal(r1.y_out, r2.y_out)
        assert r1.scal_invocations == 0 and r1.atomic_adds == 0
        assert r1.flops == 2 * 3000 * 3000 + 2 * 3000

    def test_beta_zero_kills_nan(self):
        rng = np.random.default_rng(23)
        v, _ = dev_matrix(rng, 64, 64, "d")
        got = kb.symv_hemv("u", 1.0, kb.HermitianView(v, "u"), dvec(naive.fill(rng, 64, "d")), 0.0,
                           torch.full((64,), float("nan"), device="cuda")).y_out
        assert torch.isfinite(got).all()

    def test_rejections(self):
        rng = np.random.default_rng(27)
        vc, _ = dev_matrix(rng, 32, 32, "c")
        vd, _ = dev_matrix(rng, 32, 32, "d")
        x = np.zeros(32)
        with pytest.raises(ValueError):
            kb.symv("l", 1.0, kb.HermitianView(vc, "l"), x, 0.0, x)
        with pytest.raises(ValueError):
            kb.hemv("l", 1.0, kb.HermitianView(vd, "l"), x, 0.0, x)
        with pytest.raises(ValueError):
            kb.symv_hemv("u", 1.0, kb.HermitianView(vd, "l"), x, 0.0, x)
        with pytest.raises(ValueError):
            kb.symv_hemv("l", 1.0, kb.HermitianView(vd, "l"), x, 0.0, x, hermitian=True)


class TestOffset:
    @pytest.mark.parametrize("tag", "sdcz")
    def test_paper_offsets_match_standard_bit_exact(self, tag):
        """The offset API on (i, j) of a parent == the standard API on the
        submatrix view (same realigned plan: bit-identical), and both match
        the oracle.  Offsets from BASELINE config 4 plus an aligned control."""
        rng = np.random.default_rng(31)
        parent_n = 2048
        v, a = dev_matrix(rng, parent_n, parent_n, tag)
        for (i, j) in ((1, 1), (7, 3), (13, 13), (16, 16)):
            sm, sn = parent_n - i, parent_n - j
            for trans in "nt":
                xl, yl = (sn, sm) if trans == "n" else (sm, sn)
                x, y = dvec(naive.fill(rng, xl, tag)), dvec(naive.fill(rng, yl, tag))
                off = kb.gemv_offset(trans, 1.0, kb.OffsetRequest(v, i, j, sm, sn), x, 0.5, y).y_out
                std = kb.gemv(trans, 1.0, v.submatrix(i, j, sm, sn), x, 0.5, y).y_out
                assert torch.equal(off, std)
                sa = a[i:, j:]
                want = naive.naive_gemv(trans, 1.0, sa, x.cpu().numpy(), 0.5, y.cpu().numpy())
                dense = np.abs(sa) if trans == "n" else np.abs(sa).T
                check(off, want, tag, 1.0, dense, x.cpu().numpy(), 0.5, y.cpu().numpy())
            for uplo in "lu":
                d = parent_n - i
                x, y = dvec(naive.fill(rng, d, tag)), dvec(naive.fill(rng, d, tag))
                hv = kb.HermitianView(v, uplo)
                off = kb.symv_hemv_offset(uplo, 1.0, hv, i, d, x, 0.5, y).y_out
                std = kb.symv_hemv(uplo, 1.0, kb.HermitianView(v.submatrix(i, i, d, d), uplo), x, 0.5, y).y_out
                assert torch.equal(off, std)
                sa = a[i:, i:]
                herm = tag in "cz"
                want = naive.naive_symv_hemv(1.0, sa, uplo, x.cpu().numpy(), 0.5, y.cpu().numpy())
                check(off, want, tag, 1.0, np.abs(naive.dense_from_triangle(sa, uplo, herm)), x.cpu().numpy(),
                      0.5, y.cpu().numpy())

    def test_unaligned_parent_ld_warns(self):
        v = kb.alloc_matrix(100, 100, kb.precision("d"), ld=101)
        req = kb.OffsetRequest(v, 3, 0, 32, 32)
        with pytest.warns(UserWarning, match="not segment-aligned"):
            kb.gemv_offset("n", 1.0, req, np.zeros(32), 0.0, np.zeros(32))

    def test_offset_counts_true_submatrix(self):
        rng = np.random.default_rng(47)
        v, _ = dev_matrix(rng, 256, 256, "d")
        rep = kb.symv_hemv_offset("l", 1.0, kb.HermitianView(v, "l"), 13, 100, np.zeros(100), 1.0,
                                  np.zeros(100))
        assert rep.flops == 2 * 100 * 100 + 2 * 100
        rep = kb.gemv_offset("n", 1.0, kb.OffsetRequest(v, 5, 9, 40, 40), np.zeros(40), 0.0, np.zeros(40))
        assert rep.scal_invocations == 1


class TestCAbi:
    """Direct C-ABI calls (the boundary a C/ctypes binding would use)."""

    @pytest.mark.parametrize("tag", "sdcz")
    def test_sync_and_async_entry_points(self, tag):
        lib = _lib.load()
        rng = np.random.default_rng(41)
        m, n = 777, 555
        v, a = dev_matrix(rng, m, n, tag, ld=800)
        x, y = naive.fill(rng, n, tag), naive.fill(rng, m, tag)
        xt = dvec(x)
        for suffix in ("", "_async"):
            yt = dvec(y)
            f = getattr(lib, f"kblas_{tag}gemv{suffix}")
            args = [b"N", m, n, _lib.scalar(tag, 0.25), v.data.data_ptr(), 800, xt.data_ptr(), 1,
                    _lib.scalar(tag, 2.0), yt.data_ptr(), 1]
            if suffix:
                args.append(torch.cuda.current_stream().cuda_stream)
            assert f(*args) == 0
            torch.cuda.synchronize()
            check(yt, naive.naive_gemv("n", 0.25, a, x, 2.0, y), tag, 0.25, np.abs(a), x, 2.0, y)

    def test_symv_mgpu_c_entry_single_device(self):
        """kblas_dsymv_mgpu with every logical GPU mapped to device 0."""
        lib = _lib.load()
        rng = np.random.default_rng(42)
        d, nb, G = 1000, 64, 3
        v, a = dev_matrix(rng, d, d, "d")
        dist = kb.distribute(v, nb, G)
        x, y = naive.fill(rng, d, "d"), naive.fill(rng, d, "d")
        xs = [dvec(x) for _ in range(G)]
        ys = [dvec(y)] + [torch.empty(d, dtype=torch.float64, device="cuda") for _ in range(G - 1)]
        arr = ctypes.c_void_p * G
        pa = arr(*[dist.local_views[g].data.data_ptr() for g in range(G)])
        px = arr(*[t.data_ptr() for t in xs])
        py = arr(*[t.data_ptr() for t in ys])
        ids = (ctypes.c_int * G)(*([0] * G))
        ld = dist.local_views[0].ld
        rc = lib.kblas_dsymv_mgpu(b"L", d, _lib.scalar("d", 0.5), pa, ld, px, 1, _lib.scalar("d", -1.0), py, 1,
                                  G, nb, ids)
        assert rc == 0
        want = naive.naive_symv_hemv(0.5, a, "l", x, -1.0, y)
        check(ys[0], want, "d", 0.5, np.abs(naive.dense_from_triangle(a, "l", False)), x, -1.0, y)


    def test_mgpu_async_reused_partials_back_to_back(self):
        """two kblas_dsymv_mgpu_async calls in a row on separate
        per-GPU streams reuse the same dy[g]; GPU g's stream must wait for
        the first call's root combine before its next partial overwrites
        dy[g].  A long first call (big operand, small second) makes the race
        visible if the wait were missing."""
        lib = _lib.load()
        rng = np.random.default_rng(44)
        n, G, nb = 4096, 2, 128
        arr = ctypes.c_void_p * G
        ids = (ctypes.c_int * G)(*([0] * G))
        dA = arr()
        ldda = ctypes.c_int(0)
        assert lib.kblas_malloc_mgpu_1d(n, n, 8, dA, ctypes.byref(ldda), G, nb, ids) == 0
        a = np.asfortranarray(naive.fill(rng, (n, n), "d"))
        assert lib.kblas_setmatrix_mgpu_1d(n, n, 8, a.ctypes.data, n, dA, ldda.value, G, nb, ids) == 0
        streams = [torch.cuda.Stream() for _ in range(G)]
        pst = arr(*[s_.cuda_stream for s_ in streams])
        outs, wants = [], []
        y_part = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(G - 1)]
        torch.cuda.synchronize()
        for it in range(6):
            x = naive.fill(rng, n, "d")
            xs = [dvec(x) for _ in range(G)]
            y0 = torch.zeros(n, dtype=torch.float64, device="cuda")
            py = arr(*([y0.data_ptr()] + [t.data_ptr() for t in y_part]))
            px = arr(*[t.data_ptr() for t in xs])
            rc = lib.kblas_dsymv_mgpu_async(b"L", n, 1.0, dA, ldda.value, px, 1, 0.0, py, 1, G, nb, ids, pst)
            assert rc == 0
            outs.append((y0, xs))
            wants.append(naive.naive_symv_hemv(1.0, np.tril(a), "l", x, 0.0, np.zeros(n)))
        torch.cuda.synchronize()
        dense = np.abs(naive.dense_from_triangle(np.tril(a), "l", False))
        for (y0, xs), want, in zip(outs, wants):
            check(y0, want, "d", 1.0, dense, xs[0].cpu().numpy(), 0.0, np.zeros(n))
        assert lib.kblas_free_mgpu(dA, G, ids) == 0

    @pytest.mark.parametrize("kind", ["zhemv", "sgemv_t", "dgemv_n"])
    def test_mgpu_async_c_entries_and_allocation(self, kind):
        """kblas_malloc_mgpu_1d + kblas_setmatrix_mgpu_1d + the _mgpu_async
        entry on user streams (every logical GPU on device 0), checked against
        the oracle; then kblas_free_mgpu."""
        lib = _lib.load()
        tag = kind[0]
        rng = np.random.default_rng(43)
        m = n = 700
        G = 3
        nb = lib.kblas_mgpu_block_size(tag.encode(), b"s" if "mv" in kind and "gemv" not in kind else b"g")
        assert nb == 128
        a = naive.fill(rng, (m, n), tag)
        a_f = np.asfortranarray(a)
        esize = a.dtype.itemsize
        arr = ctypes.c_void_p * G
        dA = arr()
        ldda = ctypes.c_int(0)
        ids = (ctypes.c_int * G)(*([0] * G))
        assert lib.kblas_malloc_mgpu_1d(m, n, esize, dA, ctypes.byref(ldda), G, nb, ids) == 0
        assert ldda.value == 704 and all(dA[g] for g in range(G))
        assert lib.kblas_setmatrix_mgpu_1d(m, n, esize, a_f.ctypes.data, m, dA, ldda.value, G, nb, ids) == 0
        dt = DT[tag]
        trans = kind.split("_")[1] if "_" in kind else None
        xl, yl = (n, m) if trans in (None, "n") else (m, n)
        x, y = naive.fill(rng, xl, tag), naive.fill(rng, yl, tag)
        xs = [dvec(x) for _ in range(G)]
        ys = [dvec(y)] + [torch.empty(yl, dtype=dt, device="cuda") for _ in range(G - 1)]
        streams = [torch.cuda.Stream() for _ in range(G)]
        pst = arr(*[s.cuda_stream for s in streams])
        px, py = arr(*[t.data_ptr() for t in xs]), arr(*[t.data_ptr() for t in ys])
        torch.cuda.synchronize()
        al, be = _lib.scalar(tag, 0.5), _lib.scalar(tag, -1.0)
        if kind == "zhemv":
            rc = lib.kblas_zhemv_mgpu_async(b"L", n, al, dA, ldda.value, px, 1, be, py, 1, G, nb, ids, pst)
            want = naive.naive_symv_hemv(0.5, np.tril(a), "l", x, -1.0, y, hermitian=True)
            dense = np.abs(naive.dense_from_triangle(np.tril(a), "l", True))
        else:
            f = getattr(lib, f"kblas_{tag}gemv_mgpu_async")
            rc = f(trans.encode(), m, n, al, dA, ldda.value, px, 1, be, py, 1, G, nb, ids, pst)
            want = naive.naive_gemv(trans, 0.5, a, x, -1.0, y)
            dense = np.abs(a) if trans == "n" else np.abs(a).T
        assert rc == 0
        streams[0].synchronize()
        check(ys[0], want, tag, 0.5, dense, x, -1.0, y)
        assert lib.kblas_free_mgpu(dA, G, ids) == 0
        assert not any(dA[g] for g in range(G))


class TestLarge:
    """Sizes the numpy oracle cannot hold comfortably: the streamed C oracle
    (all host threads) and size-independent properties."""

    def test_dsymv_16384_vs_streamed_oracle(self):
        d = 16384
        g = torch.Generator(device="cuda").manual_seed(5)
        A = torch.rand(d, d, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
        v = kb.view_of(A.T)  # column-major view of a row-major tensor
        x = torch.rand(d, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
        y = torch.rand(d, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
        for uplo in "lu":
            got = kb.symv_hemv(uplo, 1.0, kb.HermitianView(v, uplo), x, 0.5, y).y_out.cpu().numpy()
            a_host = v.array().cpu().numpy()
            xh, yh = x.cpu().numpy(), y.cpu().numpy()
            want = streamed.symv(uplo, 1.0, a_host, xh, 0.5, yh)
            norm = streamed.symv_norm_inf(uplo, a_host)
            bound = 50 * np.finfo(np.float64).eps * (norm * np.max(np.abs(xh)) + 0.5 * np.max(np.abs(yh)))
            assert naive.max_abs_error(got, want) <= bound

    def test_symv_equals_gemv_on_mirrored_matrix_32768(self):
        """DSYMV L at BASELINE config 2 size vs DGEMV on the explicitly mirrored
        matrix (two independent kernels), plus linearity in x."""
        d = 32768
        g = torch.Generator(device="cuda").manual_seed(6)
        A = torch.rand(d, d, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
        L = torch.tril(A)
        del A
        full = L + torch.tril(L, -1).T  # symmetric, row-major == column-major
        x1 = torch.rand(d, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
        x2 = torch.rand(d, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
        y0 = torch.zeros(d, device="cuda", dtype=torch.float64)
        lv = kb.view_of(L.T.contiguous().T)
        del L
        hv = kb.HermitianView(lv, "l")
        s1 = kb.symv_hemv("l", 1.0, hv, x1, 0.0, y0).y_out
        g1 = kb.gemv("n", 1.0, kb.view_of(full.T), x1, 0.0, y0).y_out
        bound = 50 * np.finfo(np.float64).eps * d * 1.0
        assert (s1 - g1).abs().max().item() <= bound
        s2 = kb.symv_hemv("l", 1.0, hv, x2, 0.0, y0).y_out
        s12 = kb.symv_hemv("l", 1.0, hv, x1 + x2, 0.0, y0).y_out
        assert (s12 - (s1 + s2)).abs().max().item() <= 2 * bound


@pytest.fixture(params=["tma", "regs"])
def symv_path(request):
    """Run a test on both SYMV/HEMV streaming kernels: the TMA-fed
    warp-specialised pipeline (default) and the register-load kernel."""
    prev = _lib.set_tma(request.param == "tma")
    yield request.param
    _lib.set_tma(prev)


class TestSymvBothPaths:
    @pytest.mark.parametrize("tag", "sdcz")
    @pytest.mark.parametrize("uplo", "lu")
    def test_oracle_both_paths(self, symv_path, tag, uplo):
        rng = np.random.default_rng(121)
        for d in (1, 31, 64, 129, 700, 1537):
            for ro in (0, 3):
                host = np.full((d + ro + 8) * (d + ro), np.nan, dtype=naive.DTYPES[tag])
                ld = d + ro + 8
                win = naive.window(host, ld, d + ro, d + ro)
                vals = naive.fill(rng, (d, d), tag)
                mask = np.tril(np.ones((d, d), bool)) if uplo == "l" else np.triu(np.ones((d, d), bool))
                tri = np.where(mask, vals, 0)
                sub = win[ro:, ro:]
                sub[mask] = vals[mask]
                v = kb.MatrixView(torch.from_numpy(host).cuda(), d + ro, d + ro, ld, kb.precision(tag)).submatrix(
                    ro, ro, d, d)
                x, y = naive.fill(rng, d, tag), naive.fill(rng, d, tag)
                rep = kb.symv_hemv(uplo, 0.75, kb.HermitianView(v, uplo), dvec(x), 1.25, dvec(y))
                assert ("symv_tma" in rep.plan) == (symv_path == "tma" and (ld * v.precision.element_bytes) % 16 == 0)
                herm = tag in "cz"
                want = naive.naive_symv_hemv(0.75, tri, uplo, x, 1.25, y, hermitian=herm)
                got = rep.y_out
                assert torch.isfinite(got).all()
                check(got, want, tag, 0.75, np.abs(naive.dense_from_triangle(tri, uplo, herm)), x, 1.25, y)

    def test_paths_agree_and_are_deterministic(self, symv_path):
        rng = np.random.default_rng(122)
        v, a = dev_matrix(rng, 5000, 5000, "d")
        x, y = dvec(naive.fill(rng, 5000, "d")), dvec(naive.fill(rng, 5000, "d"))
        r1 = kb.symv_hemv("l", 1.0, kb.HermitianView(v, "l"), x, 0.5, y).y_out
        r2 = kb.symv_hemv("l", 1.0, kb.HermitianView(v, "l"), x, 0.5, y).y_out
        assert torch.equal(r1, r2)
        want = streamed.symv("l", 1.0, a, x.cpu().numpy(), 0.5, y.cpu().numpy())
        check(r1, want, "d", 1.0, np.abs(naive.dense_from_triangle(a, "l", False)), x.cpu().numpy(), 0.5,
              y.cpu().numpy())


class TestGemvEpilogueModes:
    """GEMV reduces cross-CTA partials either in the streaming kernel (the
    last CTA of a row/column block sums the slots: few CTAs per block, large
    problems) or in a separate epilogue kernel (many CTAs per block, small
    problems).  Both are checked against the streamed oracle, and repeated
    calls must be bit-identical whichever CTA finishes last."""

    @pytest.mark.parametrize("tag", "dz")
    @pytest.mark.parametrize("trans", "nt")
    @pytest.mark.parametrize("shape", [(12000, 12000), (30000, 2000), (2000, 30000), (700, 900)])
    def test_fused_and_unfused(self, tag, trans, shape):
        m, n = shape
        g = torch.Generator(device="cuda").manual_seed(m + n)
        dt = DT[tag]
        A = torch.empty(n, m, dtype=dt, device="cuda")
        (torch.view_as_real(A) if A.is_complex() else A).uniform_(-1, 1, generator=g)
        v = kb.view_of(A.T)
        xl, yl = (n, m) if trans == "n" else (m, n)
        x = torch.empty(xl, dtype=dt, device="cuda")
        y = torch.empty(yl, dtype=dt, device="cuda")
        (torch.view_as_real(x) if x.is_complex() else x).uniform_(-1, 1, generator=g)
        (torch.view_as_real(y) if y.is_complex() else y).uniform_(-1, 1, generator=g)
        r1 = kb.gemv(trans, 0.5, v, x, -2.0, y)
        r2 = kb.gemv(trans, 0.5, v, x, -2.0, y)
        assert torch.equal(r1.y_out, r2.y_out)
        a_host = v.array().cpu().numpy()
        xh, yh = x.cpu().numpy(), y.cpu().numpy()
        want = streamed.gemv(trans, 0.5, a_host, xh, -2.0, yh)
        dense = np.abs(a_host) if trans == "n" else np.abs(a_host).T
        check(r1.y_out, want, tag, 0.5, dense, xh, -2.0, yh)


@pytest.fixture(params=["split", "stacked", "rowown0", "rowown2", "rowown5", "rowown7"])
def gemv_form(request):
    """Run a test on every GEMV-N form: the split form (narrow row blocks,
    CTAs of a row block reduced by the last to arrive), the stacked-rows
    stream-K form, and row-owning CTAs in several configurations (which
    fall back to the other forms when the matrix has too few rows)."""
    lib = _lib.load()
    mode = {"split": 1, "stacked": 0}.get(request.param, 3)
    prev = lib.kblas_set_gemv_split(mode)
    prev_c = lib.kblas_set_gemv_rowown(int(request.param[6:]) if mode == 3 else -1)
    yield request.param
    lib.kblas_set_gemv_rowown(prev_c)
    lib.kblas_set_gemv_split(prev)


class TestGemvNForms:
    @pytest.mark.parametrize("tag", "sdcz")
    def test_oracle_both_forms(self, gemv_form, tag):
        rng = np.random.default_rng(131)
        for m, n in [(1, 1), (7, 5), (65, 33), (100, 3000), (1000, 37), (2049, 1537), (129, 20000), (4100, 301)]:
            for ld, ro in ((-(-m // 32) * 32 + 32, 0), (m + 11, 5), (m + 40, 3)):
                host = np.full(ld * n, np.nan, dtype=naive.DTYPES[tag])
                win = naive.window(host, ld, ro + m, n)
                a = naive.fill(rng, (m, n), tag)
                win[ro:ro + m, :] = a
                v = kb.MatrixView(torch.from_numpy(host).cuda(), ro + m, n, ld, kb.precision(tag)).submatrix(
                    ro, 0, m, n)
                x, y = naive.fill(rng, n, tag), naive.fill(rng, m, tag)
                rep = kb.gemv("n", 0.7, v, dvec(x), -0.3, dvec(y))
                if gemv_form == "split":
                    assert rep.plan.startswith(("gemv_ns", "gemv_nc")), rep.plan
                eb = v.precision.element_bytes
                rows_per_cta = ({0: 4, 2: 2, 5: 4, 7: 8}[int(gemv_form[6:])] * (32 // eb)
                                if gemv_form.startswith("rowown") else 0)
                if (gemv_form.startswith("rowown") and (v.ld * eb) % 32 == 0
                        and m >= 80 * rows_per_cta):  # enough row blocks for the GPU
                    assert rep.plan.startswith("gemv_ro"), rep.plan
                got = rep.y_out
                assert torch.isfinite(got).all()
                check(got, naive.naive_gemv("n", 0.7, a, x, -0.3, y), tag, 0.7, np.abs(a), x, -0.3, y)

    def test_forms_deterministic_and_beta_zero(self, gemv_form):
        rng = np.random.default_rng(132)
        v, a = dev_matrix(rng, 3000, 4000, "d")
        x = naive.fill(rng, 4000, "d")
        ynan = torch.full((3000,), float("nan"), dtype=torch.float64, device="cuda")
        r1 = kb.gemv("n", 1.0, v, dvec(x), 0.0, ynan).y_out
        r2 = kb.gemv("n", 1.0, v, dvec(x), 0.0, ynan).y_out
        assert torch.equal(r1, r2)
        want = naive.naive_gemv("n", 1.0, a, x, 0.0, np.zeros(3000))
        check(r1, want, "d", 1.0, np.abs(a), x, 0.0, np.zeros(3000))

    def test_auto_picks_split_for_small(self):
        """Built-in rules alone: the split form for a small square matrix;
        with the built-in measured table: the row-owning form."""
        prev = _lib.set_gemv_split(-1)
        saved = tuner.table()
        try:
            rng = np.random.default_rng(133)
            v, a = dev_matrix(rng, 1024, 1024, "d")
            x, y = naive.fill(rng, 1024, "d"), naive.fill(rng, 1024, "d")
            want = naive.naive_gemv("n", 1.0, a, x, 1.0, y)
            tuner.clear()
            rep = kb.gemv("n", 1.0, v, dvec(x), 1.0, dvec(y))
            assert rep.plan.startswith(("gemv_ns", "gemv_nc")), rep.plan
            check(rep.y_out, want, "d", 1.0, np.abs(a), x, 1.0, y)
            tuner.defaults()
            rep = kb.gemv("n", 1.0, v, dvec(x), 1.0, dvec(y))
            assert rep.plan.startswith("gemv_ro"), rep.plan
            check(rep.y_out, want, "d", 1.0, np.abs(a), x, 1.0, y)
        finally:
            tuner.restore(saved)
            _lib.set_gemv_split(prev)


@pytest.fixture(params=["narrow", "mid", "wide"])
def symv_tiles(request):
    """Register SYMV/HEMV kernel shapes: narrow tiles (small operands),
    8-warp CTAs at 2 per SM (mid orders) and the wide 16-warp default."""
    lib = _lib.load()
    prev_n = _lib.set_symv_narrow((1 << 30) if request.param == "narrow" else 0)
    prev_m = lib.kblas_set_symv_mid((1 << 30) if request.param == "mid" else 0)
    prev_t = _lib.set_tma(0)
    saved = tuner.table()
    tuner.clear()  # the measured table would override the forced thresholds
    yield request.param
    tuner.restore(saved)
    _lib.set_symv_narrow(prev_n)
    lib.kblas_set_symv_mid(prev_m)
    _lib.set_tma(prev_t)


class TestSymvTiles:
    @pytest.mark.parametrize("tag", "sdcz")
    @pytest.mark.parametrize("uplo", "lu")
    def test_oracle_tiles(self, symv_tiles, tag, uplo):
        rng = np.random.default_rng(141)
        for d in (1, 33, 130, 1000, 2500):
            for ro in (0, 3):
                ld = d + ro + 8
                host = np.full(ld * (d + ro), np.nan, dtype=naive.DTYPES[tag])
                win = naive.window(host, ld, d + ro, d + ro)
                vals = naive.fill(rng, (d, d), tag)
                mask = np.tril(np.ones((d, d), bool)) if uplo == "l" else np.triu(np.ones((d, d), bool))
                tri = np.where(mask, vals, 0)
                win[ro:, ro:][mask] = vals[mask]
                v = kb.MatrixView(torch.from_numpy(host).cuda(), d + ro, d + ro, ld, kb.precision(tag)).submatrix(
                    ro, ro, d, d)
                x, y = naive.fill(rng, d, tag), naive.fill(rng, d, tag)
                rep = kb.symv_hemv(uplo, 0.75, kb.HermitianView(v, uplo), dvec(x), 1.25, dvec(y))
                herm = tag in "cz"
                want = naive.naive_symv_hemv(0.75, tri, uplo, x, 1.25, y, hermitian=herm)
                assert torch.isfinite(rep.y_out).all()
                check(rep.y_out, want, tag, 0.75, np.abs(naive.dense_from_triangle(tri, uplo, herm)), x, 1.25, y)


class TestHostVectorPath:
    """numpy x and y with an HBM-resident matrix go through one
    kblas_mv_hostvec call (H2D, kernels, D2H); results must equal the
    torch-vector path bit for bit and match the oracle."""

    @pytest.mark.parametrize("tag", "sdcz")
    def test_gemv_numpy_vectors(self, tag):
        rng = np.random.default_rng(151)
        v, a = dev_matrix(rng, 700, 450, tag, ld=704)
        for trans in "ntc":
            for beta in (0.0, -0.5):
                xl, yl = (450, 700) if trans == "n" else (700, 450)
                x, y = naive.fill(rng, xl, tag), naive.fill(rng, yl, tag)
                if beta == 0.0:
                    y = np.full(yl, np.nan, dtype=naive.DTYPES[tag])
                rep = kb.gemv(trans, 1.5, v, x, beta, y)
                assert isinstance(rep.y_out, np.ndarray) and rep.y_out.dtype == naive.DTYPES[tag]
                ref = kb.gemv(trans, 1.5, v, dvec(x), beta, dvec(y)).y_out.cpu().numpy()
                assert np.array_equal(rep.y_out, ref)
                dense = np.abs(a) if trans == "n" else np.abs(a).T
                yy = np.zeros(yl, naive.DTYPES[tag]) if beta == 0.0 else y
                check(rep.y_out, naive.naive_gemv(trans, 1.5, a, x, beta, yy), tag, 1.5, dense, x, beta, yy)

    @pytest.mark.parametrize("tag", "sdcz")
    @pytest.mark.parametrize("uplo", "lu")
    def test_symv_numpy_vectors(self, tag, uplo):
        rng = np.random.default_rng(152)
        d = 900
        v, a = dev_matrix(rng, d, d, tag)
        herm = tag in "cz"
        x, y = naive.fill(rng, d, tag), naive.fill(rng, d, tag)
        hv = kb.HermitianView(v, uplo)
        rep = kb.symv_hemv(uplo, 0.5, hv, x, 2.0, y)
        ref = kb.symv_hemv(uplo, 0.5, hv, dvec(x), 2.0, dvec(y)).y_out.cpu().numpy()
        assert np.array_equal(rep.y_out, ref)
        tri = np.tril(a) if uplo == "l" else np.triu(a)
        want = naive.naive_symv_hemv(0.5, tri, uplo, x, 2.0, y, hermitian=herm)
        check(rep.y_out, want, tag, 0.5, np.abs(naive.dense_from_triangle(tri, uplo, herm)), x, 2.0, y)
        assert rep.flops > 0 and rep.plan.startswith("symv")

    @pytest.mark.parametrize("tag", "dz")
    def test_gemv_numpy_vectors_tuned_forms(self, tag):
        """numpy x/y at orders where the built-in table selects the
        row-owning GEMV-N kernel (y written straight into the page-locked
        result) and the cluster split form."""
        rng = np.random.default_rng(155)
        for n in (2048, 4096):
            v, a = dev_matrix(rng, n, n, tag)
            for beta in (0.0, 0.75):
                x, y = naive.fill(rng, n, tag), naive.fill(rng, n, tag)
                rep = kb.gemv("n", 1.25, v, x, beta, y)
                assert rep.plan.startswith(("gemv_ro", "gemv_nc", "gemv_ns", "gemv_n ")), rep.plan
                check(rep.y_out, naive.naive_gemv("n", 1.25, a, x, beta, y), tag, 1.25, np.abs(a), x, beta, y)

    def test_result_buffers_fresh_and_recycled(self):
        """Results own their memory while alive (no aliasing between calls)
        and the page-locked buffer is reused once a result is released."""
        import gc

        rng = np.random.default_rng(154)
        v, a = dev_matrix(rng, 500, 400, "d")
        x1, x2 = naive.fill(rng, 400, "d"), naive.fill(rng, 400, "d")
        y = np.zeros(500)
        r1 = kb.gemv("n", 1.0, v, x1, 0.0, y).y_out
        keep = r1.copy()
        r2 = kb.gemv("n", 1.0, v, x2, 0.0, y).y_out
        assert r1.ctypes.data != r2.ctypes.data
        assert np.array_equal(r1, keep)  # the second call did not write into the first result
        view = r2[10:]
        ptr2 = r2.ctypes.data
        del r2
        gc.collect()
        r3 = kb.gemv("n", 1.0, v, x1, 0.0, y).y_out
        assert r3.ctypes.data != ptr2  # a view keeps the buffer alive
        assert np.array_equal(r3, keep)
        del view, r3
        gc.collect()
        r4 = kb.gemv("n", 1.0, v, x2, 0.0, y).y_out
        assert np.isfinite(r4).all()

    def test_inputs_not_mutated_and_errors(self):
        rng = np.random.default_rng(153)
        v, a = dev_matrix(rng, 300, 200, "d")
        x, y = naive.fill(rng, 200, "d"), naive.fill(rng, 300, "d")
        x0, y0 = x.copy(), y.copy()
        kb.gemv("n", 1.0, v, x, 1.0, y)
        assert np.array_equal(x, x0) and np.array_equal(y, y0)
        with pytest.raises(ValueError):
            kb.gemv("n", 1.0, v, x[:10], 1.0, y)
        with pytest.raises(ValueError):
            kb.gemv("n", 1.0, v, x, 1.0, y[:10])
        lib = _lib.load()
        one = ctypes.c_double(1.0)
        assert lib.kblas_mv_hostvec(b"d", b"q", b"n", 0, 4, 4, ctypes.addressof(one), v.data.data_ptr(), 300, 0, 0,
                                    x.ctypes.data, ctypes.addressof(one), y.ctypes.data, y.ctypes.data, None) == -2
        assert lib.kblas_mv_hostvec(b"d", b"g", b"n", 0, 4, 4, ctypes.addressof(one), v.data.data_ptr(), 300, 0, 0,
                                    None, ctypes.addressof(one), y.ctypes.data, y.ctypes.data, None) == -1


@pytest.fixture(params=["tc", "streamk"])
def gemv_t_form(request):
    """GEMV-T/C in the column-owning form (whole columns per CTA) and in
    the stream-K form (split rows, cross-CTA partials)."""
    lib = _lib.load()
    prev = lib.kblas_set_gemv_tc(1 if request.param == "tc" else 0, 0)
    yield request.param
    lib.kblas_set_gemv_tc(prev, 0)


class TestGemvTForms:
    @pytest.mark.parametrize("tag", "sdcz")
    def test_oracle_both_forms(self, gemv_t_form, tag):
        rng = np.random.default_rng(161)
        for m, n in [(1, 1), (7, 5), (65, 33), (3000, 100), (37, 1000), (2049, 1537)]:
            for ld, ro in ((-(-m // 32) * 32 + 32, 0), (m + 11, 5), (m + 40, 3)):
                host = np.full(ld * n, np.nan, dtype=naive.DTYPES[tag])
                win = naive.window(host, ld, ro + m, n)
                a = naive.fill(rng, (m, n), tag)
                win[ro:ro + m, :] = a
                v = kb.MatrixView(torch.from_numpy(host).cuda(), ro + m, n, ld, kb.precision(tag)).submatrix(
                    ro, 0, m, n)
                for trans in "tc":
                    x, y = naive.fill(rng, m, tag), naive.fill(rng, n, tag)
                    rep = kb.gemv(trans, 0.7, v, dvec(x), -0.3, dvec(y))
                    if gemv_t_form == "tc":
                        assert rep.plan.startswith("gemv_tc"), rep.plan
                    assert torch.isfinite(rep.y_out).all()
                    dense = np.abs(a).T
                    check(rep.y_out, naive.naive_gemv(trans, 0.7, a, x, -0.3, y), tag, 0.7, dense, x, -0.3, y)

    def test_mgpu_partial_tc(self, gemv_t_form):
        rng = np.random.default_rng(162)
        v, a = dev_matrix(rng, 900, 1300, "z")
        x, y = naive.fill(rng, 900, "z"), naive.fill(rng, 1300, "z")
        merged, _ = kb.gemv_mgpu("c", 1.1, kb.distribute(v, 64, 3), x, 0.4, y)
        check(merged.y_out, naive.naive_gemv("c", 1.1, a, x, 0.4, y), "z", 1.1, np.abs(a).T, x, 0.4, y)


@pytest.fixture(params=["cluster", "slots"])
def gemv_n_xcta(request):
    """Split-form GEMV-N with the cross-CTA step through a thread-block
    cluster's distributed shared memory, or through global partial slots."""
    lib = _lib.load()
    prev_s = _lib.set_gemv_split(1)
    prev_c = lib.kblas_set_gemv_cluster(1 if request.param == "cluster" else 0)
    yield request.param
    lib.kblas_set_gemv_cluster(prev_c)
    _lib.set_gemv_split(prev_s)


class TestGemvNCluster:
    @pytest.mark.parametrize("tag", "sdcz")
    def test_oracle_cluster_and_slots(self, gemv_n_xcta, tag):
        rng = np.random.default_rng(171)
        for m, n in [(65, 33), (100, 3000), (1000, 37), (2049, 1537), (700, 5000)]:
            for ld, ro in ((-(-m // 32) * 32 + 32, 0), (m + 11, 5)):
                host = np.full(ld * n, np.nan, dtype=naive.DTYPES[tag])
                win = naive.window(host, ld, ro + m, n)
                a = naive.fill(rng, (m, n), tag)
                win[ro:ro + m, :] = a
                v = kb.MatrixView(torch.from_numpy(host).cuda(), ro + m, n, ld, kb.precision(tag)).submatrix(
                    ro, 0, m, n)
                x, y = naive.fill(rng, n, tag), naive.fill(rng, m, tag)
                r1 = kb.gemv("n", 0.7, v, dvec(x), -0.3, dvec(y))
                r2 = kb.gemv("n", 0.7, v, dvec(x), -0.3, dvec(y))
                assert torch.equal(r1.y_out, r2.y_out)
                if gemv_n_xcta == "cluster" and n >= 512:
                    assert r1.plan.startswith("gemv_nc"), r1.plan
                assert torch.isfinite(r1.y_out).all()
                check(r1.y_out, naive.naive_gemv("n", 0.7, a, x, -0.3, y), tag, 0.7, np.abs(a), x, -0.3, y)

    def test_mgpu_partial_cluster(self, gemv_n_xcta):
        rng = np.random.default_rng(172)
        v, a = dev_matrix(rng, 1100, 1500, "d")
        x, y = naive.fill(rng, 1500, "d"), naive.fill(rng, 1100, "d")
        merged, _ = kb.gemv_mgpu("n", 1.1, kb.distribute(v, 64, 3), x, 0.4, y)
        check(merged.y_out, naive.naive_gemv("n", 1.1, a, x, 0.4, y), "d", 1.1, np.abs(a), x, 0.4, y)


def test_clear_cache_and_reuse():
    """kblas_clear_cache frees every cached buffer; later calls re-create
    them and give bit-identical results."""
    lib = _lib.load()
    rng = np.random.default_rng(181)
    v, a = dev_matrix(rng, 1500, 1500, "d")
    x, y = dvec(naive.fill(rng, 1500, "d")), dvec(naive.fill(rng, 1500, "d"))
    s1 = kb.symv_hemv("l", 1.0, kb.HermitianView(v, "l"), x, 0.5, y).y_out
    g1 = kb.gemv("n", 1.0, v, x, 0.5, y).y_out
    m1 = kb.symv_hemv_mgpu("l", 1.0, kb.distribute(v, 128, 2), x, 0.5, y, kb.KernelConfig(128, 2))[0].y_out
    torch.cuda.synchronize()
    assert lib.kblas_clear_cache() == 0
    s2 = kb.symv_hemv("l", 1.0, kb.HermitianView(v, "l"), x, 0.5, y).y_out
    g2 = kb.gemv("n", 1.0, v, x, 0.5, y).y_out
    m2 = kb.symv_hemv_mgpu("l", 1.0, kb.distribute(v, 128, 2), x, 0.5, y, kb.KernelConfig(128, 2))[0].y_out
    assert torch.equal(s1, s2) and torch.equal(g1, g2) and torch.equal(m1, m2)


def test_cuda_graph_capture_after_warmup():
    """After one warm-up call on a stream (which creates that stream's
    workspace and the shape's tile table), the async entry points can be
    captured into a CUDA graph and replayed: same results, no host work."""
    rng = np.random.default_rng(191)
    v, a = dev_matrix(rng, 3000, 3000, "d")
    x = dvec(naive.fill(rng, 3000, "d"))
    y = torch.empty(3000, dtype=torch.float64, device="cuda")
    g_out = torch.empty(3000, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    hv = kb.HermitianView(v, "l")
    with torch.cuda.stream(s):
        kb.symv_hemv("l", 1.0, hv, x, 0.0, y, inplace=True)
        kb.gemv("t", 1.0, v, x, 0.0, g_out, inplace=True)
        s.synchronize()
        want_s, want_g = y.clone(), g_out.clone()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            kb.symv_hemv("l", 1.0, hv, x, 0.0, y, inplace=True)
            kb.gemv("t", 1.0, v, x, 0.0, g_out, inplace=True)
    y.zero_()
    g_out.zero_()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, want_s) and torch.equal(g_out, want_g)


def test_threads_on_their_own_streams():
    """Four host threads, each on its own CUDA stream, issue device-tensor
    GEMV / SYMV calls of different shapes concurrently: workspaces and
    tile tables are per (device, stream) / per shape, so every result
    equals the same call made alone."""
    import threading

    rng = np.random.default_rng(77)
    shapes = [("d", 3000, 2000), ("z", 1500, 1500), ("s", 5000, 300), ("c", 2048, 2048)]
    cases = []
    for tag, m, n in shapes:
        v, _ = dev_matrix(rng, m, n, tag, ld=-(-m // 32) * 32)
        sq, _ = dev_matrix(rng, n, n, tag, ld=-(-n // 32) * 32)
        x, xs, y = dvec(naive.fill(rng, n, tag)), dvec(naive.fill(rng, n, tag)), dvec(naive.fill(rng, m, tag))
        herm = tag in "cz"
        want_g = kb.gemv("n", 0.5, v, x, -1.0, y).y_out
        want_s = kb.symv_hemv("l", 0.5, kb.HermitianView(sq, "l"), xs, 0.0, torch.zeros_like(xs),
                              hermitian=herm).y_out
        torch.cuda.synchronize()
        cases.append((v, sq, x, xs, y, herm, want_g, want_s))
    errors = []

    def work(t):
        v, sq, x, xs, y, herm, want_g, want_s = cases[t]
        st = torch.cuda.Stream()
        try:
            with torch.cuda.stream(st):
                for i in range(40):
                    if i % 2:
                        got = kb.symv_hemv("l", 0.5, kb.HermitianView(sq, "l"), xs, 0.0, torch.zeros_like(xs),
                                           hermitian=herm).y_out
                        want = want_s
                    else:
                        got = kb.gemv("n", 0.5, v, x, -1.0, y).y_out
                        want = want_g
                    st.synchronize()
                    if not torch.equal(got, want):
                        errors.append((t, i))
        except Exception as e:  # pragma: no cover - reported below
            errors.append((t, repr(e)))

    threads = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert errors == []
