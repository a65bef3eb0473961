"""The split SYMV/HEMV schedule (kblas_symv_kernel, run_symv): the last
~6 % of the items run as a second, programmatic-dependent grid of small
CTAs.  Its results match the one-grid schedule (KBLAS_SYMV_TAIL_PCT=0, in
a subprocess: the knob is read once) to rounding (the t2 partials are
grouped differently), the host-vector call (tail grid waiting for the
staged x) is bit-identical to the device-tensor call, and the mgpu path
uses it on every rank's panel."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import paper_1410_1726_b200 as kb
from paper_1410_1726_b200 import _lib

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1410_1726_b200 as kb
from paper_1410_1726_b200 import _lib
out = {}
for tag, d, uplo in json.loads(sys.argv[2]):
    p = kb.precision(tag)
    g = torch.Generator(device="cuda").manual_seed(d)
    A = torch.empty(d, d, dtype=p.torch_dtype, device="cuda")
    (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1, generator=g)
    x = torch.empty(d, dtype=p.torch_dtype, device="cuda")
    (torch.view_as_real(x) if p.is_complex else x).uniform_(-1, 1, generator=g)
    y = kb.symv_hemv(uplo, 1.0, kb.HermitianView(kb.view_of(A.T), uplo), x, 0.0, torch.zeros_like(x)).y_out
    yc = y.cpu().numpy()
    out[f"{tag}{d}{uplo}"] = {"plan": _lib.last_plan(), "re": np.real(yc).tolist(), "im": np.imag(yc).tolist()}
print(json.dumps(out))
"""

CASES = [("d", 20000, "l"), ("z", 16384, "u"), ("s", 40000, "l")]


def _run(env_pct):
    env = dict(os.environ)
    if env_pct is not None:
        env["KBLAS_SYMV_TAIL_PCT"] = str(env_pct)
    res = subprocess.run([sys.executable, "-c", CHILD, ROOT, json.dumps(CASES)], capture_output=True, text=True,
                         env=env, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    return json.loads(res.stdout.strip().splitlines()[-1])


def test_split_matches_one_grid():
    split, one = _run(None), _run(0)
    for tag, d, uplo in CASES:
        k = f"{tag}{d}{uplo}"
        assert "tail=0" not in split[k]["plan"] and " tail=" in split[k]["plan"], split[k]["plan"]
        assert "tail=0" in one[k]["plan"], one[k]["plan"]
        a = np.array(split[k]["re"]) + 1j * np.array(split[k]["im"])
        b = np.array(one[k]["re"]) + 1j * np.array(one[k]["im"])
        eps = kb.precision(tag).eps
        # same products, t2 partials summed in another grouping
        assert np.max(np.abs(a - b)) <= 64 * eps * np.sqrt(d) * max(1.0, np.max(np.abs(b))), k


def test_split_hostvec_bit_identical_to_device():
    d = 20000
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.empty(d, d, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=g)
    v = kb.HermitianView(kb.view_of(A.T), "l")
    hx = torch.empty(d, dtype=torch.float64, pin_memory=True).uniform_(-1, 1)
    hy = torch.empty(d, dtype=torch.float64, pin_memory=True).uniform_(-1, 1)
    for beta in (0.0, -0.5):
        got = kb.symv_hemv("l", 0.75, v, hx.numpy(), beta, hy.numpy()).y_out
        plan = _lib.last_plan()
        want = kb.symv_hemv("l", 0.75, v, hx.cuda(), beta, hy.cuda()).y_out.cpu().numpy()
        assert " tail=" in plan and "tail=0" not in plan, plan
        assert np.array_equal(got, want), beta


def test_split_mgpu_partials():
    d, nb = 24000, 128
    g = torch.Generator(device="cuda").manual_seed(6)
    A = torch.empty(d, d, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=g)
    full = kb.view_of(A.T)
    x = torch.empty(d, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=g)
    want = kb.symv_hemv("l", 1.0, kb.HermitianView(full, "l"), x, 0.0, torch.zeros_like(x)).y_out
    dist = kb.distribute(full, nb, 1, devices=[torch.device("cuda", 0)])
    got = kb.symv_hemv_mgpu("l", 1.0, dist, x, 0.0, torch.zeros_like(x), kb.KernelConfig(nb, 2))[0].y_out
    assert " tail=" in _lib.last_plan()
    err = float((got - want).abs().max() / want.abs().max())
    assert err <= 1e-12, err


def test_split_in_cuda_graph_and_threads():
    """A split call captured into a CUDA graph (programmatic edges to the
    tail grid and the epilogue) replays to the eager result; two threads
    on their own streams run split calls concurrently (per-stream tail
    counter) with unchanged results."""
    import threading

    d = 20000
    g = torch.Generator(device="cuda").manual_seed(7)
    A = torch.empty(d, d, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=g)
    hv = kb.HermitianView(kb.view_of(A.T), "l")
    x = torch.empty(d, dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=g)
    y = torch.empty(d, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        kb.symv_hemv("l", 1.0, hv, x, 0.0, y, inplace=True)
        s.synchronize()
        assert " tail=" in _lib.last_plan() and "tail=0" not in _lib.last_plan()
        want = y.clone()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            kb.symv_hemv("l", 1.0, hv, x, 0.0, y, inplace=True)
    y.zero_()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, want)

    outs, errs = [None, None], []

    def work(i):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                r = None
                for _ in range(5):
                    r = kb.symv_hemv("l", 1.0, hv, x, 0.0, torch.empty_like(x)).y_out
                st.synchronize()
                outs[i] = r
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for r in outs:
        assert torch.equal(r, want)
