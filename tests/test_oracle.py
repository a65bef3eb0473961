"""Pin the oracle against the real reference (golden vectors made by
tests/golden/make_golden.py from `blockmv`), then pin the C streamed
restatement against the numpy one.  CPU only."""

import numpy as np
import pytest

from conftest import cfg1_inputs, golden_inputs, load_golden
from oracle import blocked, naive, streamed

Z, META = load_golden()
CASES = sorted(k for k in META if k != "cfg1_dgemv_4096")


def _dense(p, flat, ld):
    return naive.window(flat, ld, p["rows"], p["cols"])


def _run_naive(p, flat, ld, x, y):
    a = _dense(p, flat, ld)
    op = p["op"]
    if op in ("gemv", "gemv_mgpu"):
        return naive.naive_gemv(p["trans"], p["alpha"], a, x, p["beta"], y)
    if op == "gemv_offset":
        sub = a[p["row_off"]:p["row_off"] + p["sub_m"], p["col_off"]:p["col_off"] + p["sub_n"]]
        return naive.naive_gemv(p["trans"], p["alpha"], sub, x, p["beta"], y)
    if op in ("symv", "symv_mgpu"):
        return naive.naive_symv_hemv(p["alpha"], a, p["uplo"], x, p["beta"], y, hermitian=p["hermitian"])
    o, s = p["offset"], p["sub_d"]
    return naive.naive_symv_hemv(p["alpha"], a[o:o + s, o:o + s], p["uplo"], x, p["beta"], y)


def _run_blocked(p, flat, ld, x, y):
    a = _dense(p, flat, ld)
    op, nb, coop = p["op"], p["nb"], p["coop"]
    if op == "gemv":
        return blocked.gemv(p["trans"], p["alpha"], a, x, p["beta"], y, nb, coop)
    if op == "gemv_offset":
        return blocked.gemv_offset(p["trans"], p["alpha"], a, p["row_off"], p["col_off"], p["sub_m"],
                                   p["sub_n"], x, p["beta"], y, nb, coop)
    if op == "symv":
        return blocked.symv_hemv(p["uplo"], p["alpha"], a, x, p["beta"], y, nb, coop, p["hermitian"])
    if op == "symv_offset":
        return blocked.symv_hemv_offset(p["uplo"], p["alpha"], a, p["offset"], p["sub_d"], x, p["beta"], y,
                                        nb, coop, p["hermitian"])
    if op == "gemv_mgpu":
        return blocked.gemv_mgpu(p["trans"], p["alpha"], a, x, p["beta"], y, p["G"], nb, coop)
    return blocked.symv_hemv_mgpu(p["uplo"], p["alpha"], a, x, p["beta"], y, p["G"], nb, coop, p["hermitian"])


@pytest.mark.parametrize("case", CASES)
def test_naive_restatement_matches_reference_oracle(case):
    """oracle/naive.py == blockmv.naive_* on the same inputs (same numpy ops:
    bit-identical on this image; a tiny tolerance covers BLAS kernel
    dispatch on another host CPU)."""
    p = META[case]
    flat, ld, x, y = golden_inputs(p)
    got = _run_naive(p, flat, ld, x, y)
    want = Z[f"{case}/naive"]
    assert got.dtype == want.dtype and got.shape == want.shape
    scale = max(1.0, float(np.max(np.abs(want))))
    assert naive.max_abs_error(got, want) <= 4 * naive.EPS[p["tag"]] * scale


@pytest.mark.parametrize("case", CASES)
def test_blocked_restatement_matches_reference_simulator(case):
    """oracle/blocked.py reproduces the reference simulator's y_out (its CPU path)."""
    p = META[case]
    flat, ld, x, y = golden_inputs(p)
    got = _run_blocked(p, flat, ld, x, y)
    want = Z[f"{case}/sim"]
    assert got.dtype == want.dtype and got.shape == want.shape
    scale = max(1.0, float(np.max(np.abs(want))))
    assert naive.max_abs_error(got, want) <= 4 * naive.EPS[p["tag"]] * scale


def test_blocked_is_bit_identical_on_this_image():
    """Same numpy calls in the same order as the reference: bit-for-bit."""
    exact = 0
    for case in CASES:
        p = META[case]
        flat, ld, x, y = golden_inputs(p)
        exact += int(np.array_equal(_run_blocked(p, flat, ld, x, y), Z[f"{case}/sim"]))
    assert exact >= 0.95 * len(CASES)


@pytest.mark.parametrize("case", [c for c in CASES if c.startswith(("gemv_", "symv_"))])
def test_streamed_c_matches_reference_oracle(case):
    """oracle/streamed.c (panel-streamed, wide precision) vs blockmv.naive_*."""
    p = META[case]
    flat, ld, x, y = golden_inputs(p)
    a = _dense(p, flat, ld)
    if p["op"] == "gemv":
        got = streamed.gemv(p["trans"], p["alpha"], a, x, p["beta"], y)
    else:
        got = streamed.symv(p["uplo"], p["alpha"], a, x, p["beta"], y, hermitian=p["hermitian"])
    want = Z[f"{case}/naive"]
    scale = max(1.0, float(np.max(np.abs(want))))
    # both accumulate in f64/c128 and round once to the operand dtype
    tol = (1.0 if p["tag"] in "sc" else 64.0) * naive.EPS[p["tag"]] * scale
    assert naive.max_abs_error(got, want) <= tol


def test_reference_counters_recorded():
    """API-visible counters of the reference: flops and scal placement."""
    for case in CASES:
        p = META[case]
        mul, add = (1, 1) if p["tag"] in "sd" else (6, 2)
        if p["op"] == "gemv":
            m, n = p["rows"], p["cols"]
            ylen = m if p["trans"] == "n" else n
            assert p["flops"] == mul * (m * n + 2 * ylen) + add * m * n
            assert p["scal_invocations"] == 1
        if p["op"] == "symv":
            d = p["rows"]
            assert p["flops"] == mul * (d * d + 2 * d) + add * d * d
            assert p["scal_invocations"] == 0


def test_cfg1_dgemv_4096_golden():
    """BASELINE config 1 (DGEMV N=4096, alpha=1, beta=0): the streamed C
    oracle and the numpy restatements reproduce the reference's outputs."""
    a, x, y = cfg1_inputs()
    want_naive = Z["cfg1_dgemv_4096/naive"]
    want_sim = Z["cfg1_dgemv_4096/sim"]
    got = streamed.gemv("n", 1.0, a, x, 0.0, y)
    assert naive.max_abs_error(got, want_naive) <= 1e-11
    assert naive.max_abs_error(naive.naive_gemv("n", 1.0, a, x, 0.0, y), want_naive) <= 1e-11
    assert naive.max_abs_error(blocked.gemv("n", 1.0, a, x, 0.0, y, 64, 1), want_sim) <= 1e-11
    bound = naive.tolerance_bound(np.abs(a), x, "d")
    assert naive.max_abs_error(want_sim, want_naive) <= bound


@pytest.mark.parametrize("tag", "sdcz")
@pytest.mark.parametrize("uplo", "lu")
def test_streamed_symv_matches_naive_midsize(tag, uplo):
    rng = np.random.default_rng(5)
    n = 1000
    a = np.asfortranarray(naive.fill(rng, (n, n), tag))
    x, y = naive.fill(rng, n, tag), naive.fill(rng, n, tag)
    got = streamed.symv(uplo, 0.5, a, x, 2.0, y, wide_out=True)
    want = naive.naive_symv_hemv(0.5, a, uplo, x, 2.0, y, out_dtype=np.complex128)
    assert np.max(np.abs(got - want)) <= 1e3 * np.finfo(np.float64).eps * n


def test_streamed_norm_inf_matches_dense():
    rng = np.random.default_rng(6)
    for tag in "dz":
        for uplo in "lu":
            a = np.asfortranarray(naive.fill(rng, (77, 77), tag))
            dense = naive.dense_from_triangle(a, uplo, tag == "z")
            want = float(np.max(np.sum(np.abs(dense), axis=1)))
            assert abs(streamed.symv_norm_inf(uplo, a) - want) <= 1e-12 * want


def test_streamed_unreferenced_triangle_never_read():
    """NaN in the unreferenced triangle must not reach the result."""
    rng = np.random.default_rng(7)
    n = 64
    for uplo in "lu":
        a = np.asfortranarray(naive.fill(rng, (n, n), "d"))
        clean = np.tril(a) if uplo == "l" else np.triu(a)
        poisoned = np.array(clean, order="F")
        mask = np.triu(np.ones((n, n), bool), 1) if uplo == "l" else np.tril(np.ones((n, n), bool), -1)
        poisoned[mask] = np.nan
        x, y = naive.fill(rng, n, "d"), naive.fill(rng, n, "d")
        got = streamed.symv(uplo, 1.0, poisoned, x, 0.0, y)
        assert np.all(np.isfinite(got))
        assert naive.max_abs_error(got, naive.naive_symv_hemv(1.0, clean, uplo, x, 0.0, y)) <= 1e-12


# ------------------------------------------------ generated operands
# oracle/gen.py + streamed.c's generated source: the large-N parity tests
# (tests/test_gpu_baseline_configs.py) never copy the operand to the host;
# both sides regenerate it from (seed, row, column).  Pin that the three
# restatements agree bit for bit and that the generated-source oracle is
# the memory-source oracle (pinned above against blockmv) on the same data.
from oracle import gen  # noqa: E402


@pytest.mark.parametrize("tag", "sdcz")
def test_generator_numpy_c_torch_bit_identical(tag):
    import torch

    for (m, n, gld, ro, co) in [(37, 23, 100, 3, 7), (64, 64, 64, 0, 0), (5, 200, 1 << 17, 99, 1 << 16)]:
        a_np = gen.matrix_np(tag, m, n, 5, gld, ro, co)
        a_c = streamed.gen_fill(tag, m, n, 5, gld, ro, co)
        t = torch.empty(n, m + 3, dtype=getattr(torch, gen.DT[tag]))
        gen.fill_columns(t, tag, 5, gld, m, 0, ro, co)
        a_t = t[:, :m].numpy().T
        assert a_np.dtype == a_c.dtype == a_t.dtype == naive.DTYPES[tag]
        assert np.array_equal(a_np, a_c) and np.array_equal(a_np, a_t)
    v = gen.vector_np(tag, 1000, 3)
    assert np.array_equal(v, gen.vector_torch(tag, 1000, 3, "cpu").numpy())
    assert np.all(np.abs(v.real) <= 1.0) and abs(float(np.mean(v.real))) < 0.1


def test_generator_triangle_poison():
    import torch

    t = torch.empty(8, 8, dtype=torch.float64)
    gen.fill_columns(t, "d", 1, 8, 8, tri="l")
    a = t.numpy().T  # a[i, c]
    assert np.all(np.isnan(a[np.triu_indices(8, 1)])) and not np.any(np.isnan(a[np.tril_indices(8)]))
    # a block of columns written on its own equals the same columns of the whole
    part = torch.empty(3, 8, dtype=torch.float64)
    gen.fill_columns(part, "d", 1, 8, 8, col0=4, tri="l")
    assert np.array_equal(part.numpy(), t.numpy()[4:7], equal_nan=True)


@pytest.mark.parametrize("tag", "sdcz")
def test_generated_oracle_equals_memory_oracle(tag):
    n, seed = 257, 9
    for off in (0, 13):
        a = streamed.gen_fill(tag, n, n, seed, n + off, off, off)
        x, y = gen.vector_np(tag, n, 10), gen.vector_np(tag, n, 11)
        for uplo in "lu":
            want = streamed.symv(uplo, 0.5, a, x, 0.25, y, nthreads=1)
            got, norm = streamed.symv_gen(tag, uplo, n, seed, n + off, off, 0.5, x, 0.25, y, nthreads=1)
            assert np.array_equal(got, want)
            assert norm == pytest.approx(streamed.symv_norm_inf(uplo, a), rel=1e-12)
            ref = naive.naive_symv_hemv(0.5, a, uplo, x, 0.25, y)
            dense = np.abs(naive.dense_from_triangle(a, uplo, tag in "cz"))
            assert naive.max_abs_error(got, ref) <= naive.run_bound(tag, 0.5, dense, x, 0.25, y)
        for trans in "ntc":
            want = streamed.gemv(trans, -1.5, a, x, 0.25, y, nthreads=1)
            got, norm = streamed.gemv_gen(tag, trans, n, n, seed, n + off, off, off, -1.5, x, 0.25, y, nthreads=1)
            assert np.array_equal(got, want)
            aw = np.abs(naive.wide(a))
            opa = aw if trans == "n" else aw.T
            assert norm == pytest.approx(float(np.max(opa.sum(axis=1))), rel=1e-12)


def test_generated_oracle_rectangular_offsets():
    """gemv_gen on an offset window equals the memory oracle on the same
    window of the materialised parent (configs[3] shape family)."""
    N, i, j = 300, 7, 3
    parent = streamed.gen_fill("z", N, N, 4, N)
    sub = parent[i:, j:]
    x_n, x_t = gen.vector_np("z", N - j, 1), gen.vector_np("z", N - i, 1)
    y_n, y_t = gen.vector_np("z", N - i, 2), gen.vector_np("z", N - j, 2)
    for trans, x, y in (("n", x_n, y_n), ("t", x_t, y_t), ("c", x_t, y_t)):
        want = streamed.gemv(trans, 1.0, sub, x, 0.5, y, nthreads=1)
        got, _ = streamed.gemv_gen("z", trans, N - i, N - j, 4, N, i, j, 1.0, x, 0.5, y, nthreads=1)
        assert np.array_equal(got, want)
