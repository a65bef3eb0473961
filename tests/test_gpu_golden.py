"""GPU parity against the reference's own outputs (golden vectors from the
real `blockmv`): every case runs through the drop-in Python API on
HBM-resident operands and must match blockmv.naive_* within the
reference's bound 50 eps (|alpha| ||A||_inf ||x||_inf + |beta| ||y||_inf)
(cli.py:171-175) and the reference simulator's y_out within the same
bound."""

import numpy as np
import pytest
import torch

import paper_1410_1726_b200 as kb
from conftest import cfg1_inputs, golden_inputs, load_golden
from oracle import naive

pytestmark = pytest.mark.gpu

Z, META = load_golden()
CASES = sorted(k for k in META if k != "cfg1_dgemv_4096")


def _dev_view(p, flat, ld):
    prec = kb.precision(p["tag"])
    t = torch.from_numpy(flat).cuda()
    return kb.MatrixView(t, p["rows"], p["cols"], ld, prec)


def _bound(p, dense_abs, x, y):
    return naive.run_bound(p["tag"], p["alpha"], dense_abs, x, p["beta"], y)


@pytest.mark.parametrize("case", CASES)
def test_golden_case(case):
    p = META[case]
    flat, ld, x, y = golden_inputs(p)
    v = _dev_view(p, flat, ld)
    a_host = naive.window(flat, ld, p["rows"], p["cols"])
    op = p["op"]
    xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    if op == "gemv":
        got = kb.gemv(p["trans"], p["alpha"], v, xt, p["beta"], yt).y_out
        dense = np.abs(a_host)
    elif op == "gemv_offset":
        req = kb.OffsetRequest(v, p["row_off"], p["col_off"], p["sub_m"], p["sub_n"])
        got = kb.gemv_offset(p["trans"], p["alpha"], req, xt, p["beta"], yt).y_out
        dense = np.abs(a_host[p["row_off"]:p["row_off"] + p["sub_m"], p["col_off"]:p["col_off"] + p["sub_n"]])
    elif op == "symv":
        hv = kb.HermitianView(v, p["uplo"])
        got = kb.symv_hemv(p["uplo"], p["alpha"], hv, xt, p["beta"], yt, hermitian=p["hermitian"]).y_out
        dense = np.abs(naive.dense_from_triangle(a_host, p["uplo"], p["hermitian"]))
    elif op == "symv_offset":
        hv = kb.HermitianView(v, p["uplo"])
        got = kb.symv_hemv_offset(p["uplo"], p["alpha"], hv, p["offset"], p["sub_d"], xt, p["beta"], yt).y_out
        o, s = p["offset"], p["sub_d"]
        dense = np.abs(naive.dense_from_triangle(a_host[o:o + s, o:o + s], p["uplo"], p["hermitian"]))
    elif op == "gemv_mgpu":
        dist = kb.distribute(v, p["nb"], p["G"])
        got = kb.gemv_mgpu(p["trans"], p["alpha"], dist, xt, p["beta"], yt)[0].y_out
        dense = np.abs(a_host)
    else:
        dist = kb.distribute(v, p["nb"], p["G"])
        got = kb.symv_hemv_mgpu(p["uplo"], p["alpha"], dist, xt, p["beta"], yt,
                                kb.KernelConfig(p["nb"], 2))[0].y_out
        dense = np.abs(naive.dense_from_triangle(a_host, p["uplo"], p["hermitian"]))
    got = got.cpu().numpy()
    want = Z[f"{case}/naive"]
    sim = Z[f"{case}/sim"]
    if op in ("gemv", "gemv_offset", "gemv_mgpu") and p["trans"] != "n":
        dense = dense.T
    bound = _bound(p, dense, x, y)
    assert got.dtype == want.dtype and got.shape == want.shape
    assert np.all(np.isfinite(got))
    assert naive.max_abs_error(got, want) <= bound, case
    assert naive.max_abs_error(got, sim) <= 2 * bound, case


def test_cfg1_dgemv_4096():
    """BASELINE config 1 through the drop-in API vs the reference's outputs."""
    a, x, y = cfg1_inputs()
    v = kb.view_of(torch.from_numpy(np.ascontiguousarray(a.T)).cuda().T)
    got = kb.gemv("n", 1.0, v, torch.from_numpy(x).cuda(), 0.0, torch.from_numpy(y).cuda()).y_out.cpu().numpy()
    bound = naive.tolerance_bound(np.abs(a), x, "d")
    assert naive.max_abs_error(got, Z["cfg1_dgemv_4096/naive"]) <= bound
    assert naive.max_abs_error(got, Z["cfg1_dgemv_4096/sim"]) <= bound


def test_cfg1_host_buffers_roundtrip():
    """Same config through host numpy operands (the e2e path): numpy in, numpy out."""
    a, x, y = cfg1_inputs()
    v = kb.view_of(a)
    rep = kb.gemv("n", 1.0, v, x, 0.0, y)
    assert isinstance(rep.y_out, np.ndarray)
    bound = naive.tolerance_bound(np.abs(a), x, "d")
    assert naive.max_abs_error(rep.y_out, Z["cfg1_dgemv_4096/naive"]) <= bound
    assert rep.flops == META["cfg1_dgemv_4096"]["flops"]
    assert rep.scal_invocations == 1
