"""Host-side logic of the drop-in (no GPU needed): argument types and
validation mirrored from the reference, layout/partition arithmetic, the
algorithmic byte/flop counts, and the C-ABI library surface."""

import ctypes
import os

import numpy as np
import pytest

from paper_1410_1726_b200 import _lib, roofline
from paper_1410_1726_b200.core import HermitianView, MatrixView, precision, view_of
from paper_1410_1726_b200.multidevice import (
    local_col_count,
    owned_block_cols,
    required_local_elements,
)
from paper_1410_1726_b200.offset import OffsetRequest, effective_dims, realigned_frame
from paper_1410_1726_b200.partition import KernelConfig, sk_owner, sk_start, tb_share


class TestPrecision:
    def test_tags(self):
        assert precision("D").element_bytes == 8
        assert precision("z").flops_per_mul == 6 and precision("z").flops_per_add == 2
        with pytest.raises(ValueError):
            precision("q")

    def test_eps_of_real_component(self):
        assert precision("c").eps == np.finfo(np.float32).eps
        assert precision("z").eps == np.finfo(np.float64).eps


class TestViews:
    def test_matrix_view_validation(self):
        prec = precision("d")
        buf = np.zeros(100, dtype=np.float64)
        with pytest.raises(ValueError):
            MatrixView(buf, 0, 3, 10, prec)
        with pytest.raises(ValueError):
            MatrixView(buf, 10, 3, 9, prec)  # ld too small
        with pytest.raises(ValueError):
            MatrixView(buf, 10, 11, 10, prec)  # buffer too small
        with pytest.raises(ValueError):
            MatrixView(buf.astype(np.float32), 10, 3, 10, prec)  # dtype

    def test_linear_index_and_submatrix(self):
        prec = precision("s")
        buf = np.arange(64, dtype=np.float32)
        v = MatrixView(buf, 8, 8, 8, prec)
        sub = v.submatrix(2, 3, 4, 5)
        assert sub.linear_index(0, 0) == 3 * 8 + 2
        assert sub.array()[1, 2] == buf[(3 + 2) * 8 + 2 + 1]
        assert v.decode_linear(sub.linear_index(1, 2)) == (3, 5)
        with pytest.raises(ValueError):
            v.submatrix(5, 0, 4, 1)

    def test_view_of_fortran_array(self):
        a = np.asfortranarray(np.arange(12, dtype=np.float64).reshape(3, 4))
        v = view_of(a)
        assert v.rows == 3 and v.cols == 4 and np.array_equal(v.array(), a)

    def test_hermitian_view(self):
        v = MatrixView(np.zeros(16), 4, 4, 4, precision("d"))
        hv = HermitianView(v, "L")
        assert hv.uplo == "l" and hv.dim == 4
        with pytest.raises(ValueError):
            HermitianView(v, "x")
        with pytest.raises(ValueError):
            HermitianView(MatrixView(np.zeros(16), 4, 3, 4, precision("d")), "l")


class TestPartition:
    def test_kernel_config_validation(self):
        KernelConfig(32, 4, 2)
        for bad in ((31, 1), (0, 1), (32, 0), (32, 3)):
            with pytest.raises(ValueError):
                KernelConfig(*bad)
        with pytest.raises(ValueError):
            KernelConfig(32, 2, 0)

    def test_tb_share_covers(self):
        for total in range(0, 60):
            for coop in range(1, 9):
                cover = []
                for s in range(coop):
                    w, st = tb_share(total, coop, s)
                    cover.extend(range(st, st + w))
                assert cover == list(range(total))

    def test_stream_k_split(self):
        """Every item owned by exactly one CTA; shares differ by at most one."""
        for total in (1, 7, 148, 1000, 2049):
            for P in (1, 3, 148, 296):
                if P > total:
                    continue
                sizes = [sk_start(c + 1, total, P) - sk_start(c, total, P) for c in range(P)]
                assert sum(sizes) == total and max(sizes) - min(sizes) <= 1
                for i in range(0, total, max(1, total // 50)):
                    c = sk_owner(i, total, P)
                    assert sk_start(c, total, P) <= i < sk_start(c + 1, total, P)


class TestOffsetGeometry:
    def test_effective_dims(self):
        assert effective_dims(1000, 1000, 100, 70, 32) == (128, 96)
        assert effective_dims(100, 100, 97, 99, 32) == (100, 100)
        with pytest.raises(ValueError):
            effective_dims(50, 50, 51, 10, 32)

    def test_offset_request_validation(self):
        parent = MatrixView(np.zeros(64 * 64), 64, 64, 64, precision("d"))
        with pytest.raises(ValueError):
            OffsetRequest(parent, -1, 0, 8, 8)
        with pytest.raises(ValueError):
            OffsetRequest(parent, 60, 0, 8, 8)

    def test_realignment_padding_below_one_granule(self):
        for eb in (4, 8, 16):
            per = 32 // eb
            for off in range(0, 40):
                start, frame, lead = realigned_frame(off, 100, eb)
                assert start % per == 0 and 0 <= lead < per and frame == lead + 100


class TestLayout:
    def test_cyclic_ownership(self):
        assert owned_block_cols(7 * 32, 32, 3, 0) == [0, 3, 6]
        assert owned_block_cols(7 * 32, 32, 3, 1) == [1, 4]

    def test_local_counts(self):
        assert local_col_count(100, 32, 2, 0) == 64
        assert local_col_count(100, 32, 2, 1) == 36
        assert required_local_elements(100, 100, 32, 2, 0) == 128 * 64
        assert required_local_elements(100, 100, 32, 4, 3) == 128 * 4


class TestRoofline:
    def test_baseline_bytes(self):
        """The algorithmic divisors quoted in BASELINE.md §2."""
        d = precision("d")
        z = precision("z")
        assert roofline.byte_count(d, "gemv", 4096) == 134_316_032
        assert roofline.flop_count(d, "gemv", 4096) == 33_562_624
        assert roofline.byte_count(d, "symv", 32768) == 4_295_884_800
        assert roofline.flop_count(d, "symv", 32768) == 2_147_549_184
        assert roofline.byte_count(d, "symv", 100_000) == 40_002_800_000
        assert roofline.byte_count(z, "symv", 100_000) == 80_005_600_000

    def test_rectangular_forms_reduce_to_square(self):
        for tag in "sdcz":
            p = precision(tag)
            assert roofline.gemv_bytes(p, 300, 300) == roofline.byte_count(p, "gemv", 300)
            assert roofline.symv_bytes(p, 300) == roofline.byte_count(p, "symv", 300)
            assert roofline.gemv_flops(p, 300, 300) == roofline.flop_count(p, "gemv", 300)
            assert roofline.symv_flops(p, 300) == roofline.flop_count(p, "symv", 300)


class TestCAbi:
    def test_library_exports_every_header_symbol(self):
        lib = _lib.load()
        syms = _lib.header_symbols()
        assert len(syms) >= 60
        missing = [s for s in syms if not hasattr(lib, s)]
        assert missing == []

    def test_version_and_host_helpers(self):
        lib = _lib.load()
        assert b"sm_100a" in lib.kblas_version()
        assert lib.kblas_mgpu_local_cols(100, 32, 2, 1) == 36
        assert lib.kblas_mgpu_local_cols(100, 32, 4, 3) == 4
        assert lib.kblas_mgpu_local_ld(100) == 128
        assert lib.kblas_mgpu_local_cols(100, 0, 2, 1) == -1

    def test_argument_errors_are_blas_style(self):
        """xerbla numbering, checked before any device work."""
        lib = _lib.load()
        one = _lib.scalar("d", 1.0)
        assert lib.kblas_dgemv(b"x", 4, 4, one, None, 4, None, 1, one, None, 1) == -1
        assert lib.kblas_dgemv(b"n", -1, 4, one, None, 4, None, 1, one, None, 1) == -2
        assert lib.kblas_dgemv(b"n", 4, -1, one, None, 4, None, 1, one, None, 1) == -3
        assert lib.kblas_dgemv(b"n", 4, 4, one, None, 3, None, 1, one, None, 1) == -6
        assert lib.kblas_dgemv(b"n", 4, 4, one, None, 4, None, 2, one, None, 1) == -8
        assert lib.kblas_dgemv(b"n", 4, 4, one, None, 4, None, 1, one, None, 2) == -11
        assert lib.kblas_dsymv(b"q", 4, one, None, 4, None, 1, one, None, 1) == -1
        assert lib.kblas_dsymv(b"l", 4, one, None, 3, None, 1, one, None, 1) == -5
        assert lib.kblas_dsymv(b"l", 4, one, None, 4, None, 3, one, None, 1) == -7
        # quick returns: nothing to do, nothing launched
        before = lib.kblas_launch_count()
        assert lib.kblas_dgemv(b"n", 0, 0, one, None, 1, None, 1, one, None, 1) == 0
        zero = _lib.scalar("d", 0.0)
        assert lib.kblas_dsymv(b"l", 8, zero, None, 8, None, 1, one, None, 1) == 0
        assert lib.kblas_launch_count() == before

    def test_compute_without_gpu_fails_loudly(self):
        """On a host without a GPU a compute call returns a CUDA error code
        (no silent CPU path)."""
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
        lib = _lib.load()
        one = _lib.scalar("d", 1.0)
        buf = (ctypes.c_double * 64)()
        rc = lib.kblas_dgemv(b"n", 8, 8, one, ctypes.addressof(buf), 8, ctypes.addressof(buf), 1, one,
                             ctypes.addressof(buf), 1)
        assert rc > 0
        from paper_1410_1726_b200 import gemv

        with pytest.raises(RuntimeError):
            gemv("n", 1.0, MatrixView(np.zeros(64), 8, 8, 8, precision("d")), np.zeros(8), 0.0, np.zeros(8))


def test_view_of_padded_column_major_tensor():
    """a padded column-major torch tensor (ld > rows) is accepted
    when its storage holds n whole columns (the reference's rule,
    core.py:92-94)."""
    import torch

    import paper_1410_1726_b200 as kb

    t = torch.zeros(4, 10).T[:6]  # 6 x 4, ld 10
    v = kb.view_of(t)
    assert (v.rows, v.cols, v.ld) == (6, 4, 10)
    assert v.data.numel() == 40
    t[2, 3] = 5.0
    assert float(v.array()[2, 3]) == 5.0


class TestHostcallBinding:
    """csrc/kblas_hostcall.cpp: the CPython fast path of the numpy-vector
    call.  Off-path operands come back as SLOW_PATH before any device
    work, so the Python layer can convert and validate them."""

    def test_shares_the_ctypes_library_instance(self):
        from paper_1410_1726_b200 import _ops

        _lib.load()
        assert _ops.hostcall().last_plan() == _lib.last_plan()
        maps = [ln.split() for ln in open("/proc/self/maps") if "libkblas_b200.so" in ln]
        assert maps, "libkblas_b200.so is not mapped"
        assert sum(1 for f in maps if int(f[2], 16) == 0) == 1  # one load of the file

    @pytest.mark.parametrize("x, alpha, y", [
        ([1.0, 2.0, 3.0, 4.0], 1.0, np.zeros(4)),             # x is a list
        (np.zeros(4, np.float32), 1.0, np.zeros(4)),          # wrong dtype
        (np.zeros(5), 1.0, np.zeros(4)),                      # wrong length
        (np.zeros((4, 8))[:, 0], 1.0, np.zeros(4)),           # strided
        (np.zeros((2, 2)), 1.0, np.zeros(4)),                 # 2-D
        (np.zeros(4), 1j, np.zeros(4)),                       # complex alpha, real precision
        (np.zeros(4), 1.0, np.zeros(3)),                      # y length (beta == 0)
    ])
    def test_off_path_operands(self, x, alpha, y):
        from paper_1410_1726_b200 import _ops

        hc = _ops.hostcall()
        assert hc.mv_hostvec("d", "g", "n", 0, 4, 4, alpha, 0, 4, 0, 0, x, 4, 0.0, y, 4, 0, 0, True) == hc.SLOW_PATH

    def test_beta_nonzero_checks_y_dtype(self):
        from paper_1410_1726_b200 import _ops

        hc = _ops.hostcall()
        y32 = np.zeros(4, np.float32)
        assert hc.mv_hostvec("d", "g", "n", 0, 4, 4, 1.0, 0, 4, 0, 0, np.zeros(4), 4, 0.5, y32, 4, 0, 0,
                             True) == hc.SLOW_PATH

    def test_slow_path_validation_messages(self):
        """The slow path raises the reference's exceptions (kernels.py:395-399)."""
        from paper_1410_1726_b200 import _ops

        p = precision("d")
        with pytest.raises(ValueError, match="x must be a vector of length 4"):
            _ops._hostvec_operands(p, np.zeros(5), 4, 1.0, 0.0, np.zeros(4), 4, np.zeros(4))
        with pytest.raises(ValueError, match="y must be a vector of length 4"):
            _ops._hostvec_operands(p, np.zeros(4), 4, 1.0, 0.0, np.zeros(3), 4, np.zeros(4))
        with pytest.raises(ValueError, match="complex scalar"):
            _ops._hostvec_operands(p, np.zeros(4), 4, 1j, 0.0, np.zeros(4), 4, np.zeros(4))
        xa, a, b, ya = _ops._hostvec_operands(p, [1, 2, 3, 4], 4, 2, 0.5, [1, 1, 1, 1], 4, None)
        assert xa.dtype == np.float64 and ya.dtype == np.float64 and (a, b) == (2.0, 0.5)


def test_deferred_report_behaves_like_execution_report():
    """The numpy-vector path's report fills its counters on first access and
    otherwise behaves as the reference's ExecutionReport (kernels.py:37-62):
    equality, absorb, pickle, copy and dataclasses.replace."""
    import copy
    import dataclasses
    import pickle

    from paper_1410_1726_b200.kernels import ExecutionReport, _DeferredReport

    calls = []

    def fill():
        calls.append(1)
        r = ExecutionReport()
        r.bytes_read, r.flops, r.plan, r.scal_invocations = 40, 7, "gemv_ro d", 1
        return r

    d = _DeferredReport(np.arange(3.0), fill)
    assert calls == []
    assert d.flops == 7 and d.bytes_read == 40 and d.plan == "gemv_ro d" and calls == [1]
    assert d == ExecutionReport(y_out=d.y_out, bytes_read=40, flops=7, plan="gemv_ro d", scal_invocations=1)
    tot = ExecutionReport()
    tot.absorb(_DeferredReport(None, fill))
    assert tot.bytes_read == 40 and tot.scal_invocations == 1
    p = pickle.loads(pickle.dumps(_DeferredReport(np.zeros(2), fill)))
    assert type(p) is ExecutionReport and p.flops == 7
    assert copy.deepcopy(_DeferredReport(None, fill)).bytes_read == 40
    r = dataclasses.replace(_DeferredReport(None, fill), flops=9)
    assert r.flops == 9 and r.bytes_read == 40
    w = _DeferredReport(None, fill)
    w.flops += 1
    assert w.flops == 8 and w.bytes_read == 40


def test_no_noncoherent_x_loads_before_griddepcontrol_wait():
    """A main kernel launched as the programmatic dependent of the
    host-vector copy-in grid may read x only after griddepcontrol.wait.
    ptxas hoists ld.global.nc loads above the wait (SASS LDG.E.CONSTANT
    ahead of ACQBULK), so x is read with coherent loads (kblas_device.cuh
    ld_x / ld_xvec); this checks the shipped SASS: before ACQBULK the only
    non-coherent loads are the A stream's (.NA, L1::no_allocate)."""
    import re
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", _lib.LIB_PATH], capture_output=True, text=True, check=True).stdout
    checked, bad = 0, []
    for fn in re.split(r"\n\s+Function : ", sass)[1:]:
        if "ACQBULK" not in fn:
            continue
        checked += 1
        name = fn.split("\n", 1)[0].strip()
        for op in re.findall(r"LDG\.[A-Z0-9.]+", fn[: fn.index("ACQBULK")]):
            if "CONSTANT" in op and ".NA" not in op:
                bad.append((name[:80], op))
    assert checked >= 100, checked
    assert bad == [], bad[:5]


def test_hostvec_copy_in_stores_only_after_griddepcontrol_wait():
    """The host-vector copy-in grid is launched as a programmatic dependent
    of the stream's previous kernel, which may still read the staging
    buffer: it may read host memory before griddepcontrol.wait but must
    not store before it (shipped SASS: no STG ahead of ACQBULK)."""
    import re
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", _lib.LIB_PATH], capture_output=True, text=True, check=True).stdout
    fns = [f for f in re.split(r"\n\s+Function : ", sass)[1:] if f.startswith("_ZN2kb23kblas_hostvec_in_kernel")]
    assert fns  # one static copy per translation unit
    for fn in fns:
        assert "ACQBULK" in fn and "PREEXIT" in fn
        head = fn[: fn.index("ACQBULK")]
        assert re.findall(r"STG\.", head) == []
        assert re.findall(r"LDG\.E\.128", head), "the first 16-byte host reads are issued before the wait"


def test_kernel_request_validation():
    """KernelRequest keeps the reference's checks and messages
    (kernels.py:74-89)."""
    import paper_1410_1726_b200 as kb

    v = MatrixView(np.zeros(12), 3, 4, 3, precision("d"))
    cfg = kb.KernelConfig(64, 4)
    kb.KernelRequest(kb.Op.GEMV_N, v, np.zeros(4), np.zeros(3), 1.0, 0.0, cfg)
    kb.KernelRequest(kb.Op.GEMV_T, v, np.zeros(3), np.zeros(4), 1.0, 0.0, cfg)
    with pytest.raises(ValueError, match="x has length 3, expected 4"):
        kb.KernelRequest(kb.Op.GEMV_N, v, np.zeros(3), np.zeros(3), 1.0, 0.0, cfg)
    with pytest.raises(ValueError, match="y has length 4, expected 3"):
        kb.KernelRequest(kb.Op.GEMV_N, v, np.zeros(4), np.zeros(4), 1.0, 0.0, cfg)
    with pytest.raises(ValueError, match="symmetric ops need a square matrix, got 3x4"):
        kb.KernelRequest(kb.Op.SYMV_LOWER, v, np.zeros(4), np.zeros(4), 1.0, 0.0, cfg)
    sq = MatrixView(np.zeros(9), 3, 3, 3, precision("d"))
    with pytest.raises(ValueError, match="require a HermitianView"):
        kb.KernelRequest(kb.Op.SYMV_LOWER, sq, np.zeros(3), np.zeros(3), 1.0, 0.0, cfg)
    r = kb.KernelRequest(kb.Op.SYMV_LOWER, kb.HermitianView(sq, "l"), np.zeros(3), np.zeros(3), 1.0, 0.0, cfg)
    assert r.view is sq and r.precision.tag == "d"


class TestIntDimensions:
    """The C ABI's dimensions are 32-bit ints (BLAS convention); anything
    larger is rejected before a call instead of wrapping in ctypes."""

    def test_c_int_dims(self):
        from paper_1410_1726_b200 import _ops

        _ops.c_int_dims("gemv", m=2**31 - 1, n=5)
        with pytest.raises(ValueError, match=r"gemv: m = 2147483648 exceeds the C ABI's 32-bit int range"):
            _ops.c_int_dims("gemv", m=2**31, n=5)

    def test_call_sites_reject_before_any_device_work(self):
        import torch

        from paper_1410_1726_b200 import _ops

        p = precision("d")
        v = torch.zeros(4, dtype=torch.float64)
        with pytest.raises(ValueError, match="lda = 3000000000"):
            _ops.call_gemv(p, "n", 4, 4, 1.0, 0, 3_000_000_000, v, 0.0, v, "cpu")
        with pytest.raises(ValueError, match="n = 2147483648"):
            _ops.call_symv(p, False, "l", 2**31, 1.0, 0, 2**31, v, 0.0, v, "cpu")
        hc = _ops.hostcall()  # the numpy-vector path: checked in the CPython binding
        with pytest.raises(ValueError, match="32-bit int range"):
            hc.mv_hostvec("d", "g", "n", 0, 2**31, 4, 1.0, 0, 2**31, 0, 0, np.zeros(4), 4, 0.0, np.zeros(2**0), 1,
                          0, 0, True)
