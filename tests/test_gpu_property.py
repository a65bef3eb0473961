"""Property-based parity (hypothesis): random shapes, leading dimensions,
submatrix offsets, scalars and precisions through the public API against
the CPU oracle, for every GEMV-N form the dispatcher can pick (built-in
rules, tuning table, forced row-owning) and for SYMV/HEMV.  Complements
the fixed-shape tests with the combinations nobody thought to write down
(the reference's test_acceptance.py c1 sweep does the same on its
simulator)."""

import os

import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, example, given, settings
from hypothesis import strategies as st

import paper_1410_1726_b200 as kb
from oracle import naive
from paper_1410_1726_b200 import _lib

pytestmark = pytest.mark.gpu

# KB_HYP_EXAMPLES / KB_HYP_RANDOM=1: longer, randomised stress runs
SETTINGS = settings(max_examples=int(os.environ.get("KB_HYP_EXAMPLES", 150)), deadline=None,
                    derandomize=not os.environ.get("KB_HYP_RANDOM"),
                    suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])


def _view(rng, m, n, tag, pad, ro, co):
    ld = ro + m + pad
    host = np.full(ld * (co + n), np.nan, dtype=naive.DTYPES[tag])
    win = naive.window(host, ld, ro + m, co + n)
    a = naive.fill(rng, (m, n), tag)
    win[ro:ro + m, co:co + n] = a
    v = kb.MatrixView(torch.from_numpy(host).cuda(), ro + m, co + n, ld, kb.precision(tag)).submatrix(ro, co, m, n)
    return v, a


def _bound(tag, alpha, dense_abs, x, beta, y):
    return naive.run_bound(tag, alpha, dense_abs, x, beta, y)


@SETTINGS
@given(tag=st.sampled_from("sdcz"), m=st.integers(1, 5000), n=st.integers(1, 3000), pad=st.integers(0, 40),
       ro=st.integers(0, 9), co=st.integers(0, 3), trans=st.sampled_from("ntc"),
       form=st.sampled_from(["rules", "rowown", "split", "stacked"]),
       alpha=st.sampled_from([1.0, -0.5, 2.25]), beta=st.sampled_from([0.0, 1.0, -0.75]),
       seed=st.integers(0, 2 ** 16))
@example(tag="z", m=4100, n=2049, pad=7, ro=3, co=1, trans="n", form="rowown", alpha=-0.5, beta=1.0, seed=1)
@example(tag="s", m=5000, n=3000, pad=0, ro=0, co=0, trans="n", form="rules", alpha=1.0, beta=0.0, seed=2)
@example(tag="d", m=3000, n=4999, pad=33, ro=5, co=2, trans="c", form="rules", alpha=2.25, beta=-0.75, seed=3)
@example(tag="c", m=2048, n=2048, pad=0, ro=0, co=0, trans="n", form="split", alpha=1.0, beta=1.0, seed=4)
def test_gemv_any_form_matches_oracle(tag, m, n, pad, ro, co, trans, form, alpha, beta, seed):
    lib = _lib.load()
    rng = np.random.default_rng(seed)
    v, a = _view(rng, m, n, tag, pad, ro, co)
    xl, yl = (n, m) if trans == "n" else (m, n)
    x, y = naive.fill(rng, xl, tag), naive.fill(rng, yl, tag)
    mode = {"rules": -1, "rowown": 3, "split": 1, "stacked": 0}[form]
    prev = lib.kblas_set_gemv_split(mode)
    try:
        rep = kb.gemv(trans, alpha, v, torch.from_numpy(x).cuda(), beta, torch.from_numpy(y).cuda())
    finally:
        lib.kblas_set_gemv_split(prev)
    got = rep.y_out.cpu().numpy()
    want = naive.naive_gemv(trans, alpha, a, x, beta, y)
    dense = np.abs(a) if trans == "n" else np.abs(a).T
    assert np.all(np.isfinite(got)), rep.plan
    assert naive.max_abs_error(got, want) <= _bound(tag, alpha, dense, x, beta, y), rep.plan


@SETTINGS
@given(tag=st.sampled_from("sdcz"), d=st.integers(1, 3000), pad=st.integers(0, 40), off=st.integers(0, 9),
       uplo=st.sampled_from("lu"), herm=st.booleans(), alpha=st.sampled_from([1.0, -0.5]),
       beta=st.sampled_from([0.0, 0.5]), seed=st.integers(0, 2 ** 16))
@example(tag="z", d=3000, pad=5, off=3, uplo="l", herm=True, alpha=-0.5, beta=0.5, seed=1)
@example(tag="s", d=2999, pad=0, off=0, uplo="u", herm=False, alpha=1.0, beta=0.0, seed=2)
def test_symv_hemv_matches_oracle(tag, d, pad, off, uplo, herm, alpha, beta, seed):
    herm = herm and tag in "cz"
    rng = np.random.default_rng(seed)
    ld = off + d + pad
    host = np.full(ld * (off + d), np.nan, dtype=naive.DTYPES[tag])
    win = naive.window(host, ld, off + d, off + d)
    vals = naive.fill(rng, (d, d), tag)
    mask = np.tril(np.ones((d, d), bool)) if uplo == "l" else np.triu(np.ones((d, d), bool))
    tri = np.where(mask, vals, 0)
    win[off:, off:][mask] = vals[mask]  # the other triangle stays NaN: it must never be read
    v = kb.MatrixView(torch.from_numpy(host).cuda(), off + d, off + d, ld, kb.precision(tag)).submatrix(
        off, off, d, d)
    x, y = naive.fill(rng, d, tag), naive.fill(rng, d, tag)
    rep = kb.symv_hemv(uplo, alpha, kb.HermitianView(v, uplo), torch.from_numpy(x).cuda(), beta,
                       torch.from_numpy(y).cuda(), hermitian=herm)
    got = rep.y_out.cpu().numpy()
    want = naive.naive_symv_hemv(alpha, tri, uplo, x, beta, y, hermitian=herm)
    dense = np.abs(naive.dense_from_triangle(tri, uplo, herm))
    assert np.all(np.isfinite(got)), rep.plan
    assert naive.max_abs_error(got, want) <= _bound(tag, alpha, dense, x, beta, y), rep.plan
