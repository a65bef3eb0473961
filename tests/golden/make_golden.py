"""Generate golden vectors by running the REAL reference (`blockmv`) in this
container:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/blockmv_golden.npz.  Each case is generated from its
own seed with oracle/naive.py's generators (restatements of the
reference's test helpers, test_kernels.py:16-36), so the fixture stores
only the seed, shapes and parameters plus the outputs: the reference
simulator's y_out (its CPU path), the reference oracle's naive_* result
and the API-visible counters (flops, scal_invocations).  tests/ regenerate
the inputs from the seed and check the regenerated A/x/y against stored
checksums before comparing.
The large DGEMV N=4096 case (BASELINE config 1) stores only y: its A, x
are regenerated from the cli.py recipe (default_rng(0), A -> x -> y).
/root/reference is read-only and absent on the GPU box, so only this
script touches it; tests read the .npz.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import naive  # noqa: E402
import blockmv  # noqa: E402
from blockmv.core import HermitianView, make_padded_view, precision  # noqa: E402
from blockmv.partition import KernelConfig  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "blockmv_golden.npz")
store: dict = {}
meta: dict = {}


_seed = [1000]


def case_inputs(m, n, xl, yl, tag):
    """Seeded inputs: A (m x n, ld padded to 32), x, y from oracle.naive."""
    _seed[0] += 1
    rng = np.random.default_rng(_seed[0])
    flat, ld = naive.random_matrix(rng, m, n, tag)
    x, y = naive.random_vec(rng, xl, tag), naive.random_vec(rng, yl, tag)
    v = blockmv.MatrixView(data=flat, rows=m, cols=n, ld=ld, precision=precision(tag))
    return _seed[0], v, x, y


def checksum(a) -> float:
    a = np.asarray(a)
    return float(np.sum(np.abs(a.astype(np.complex128)) * np.arange(1, a.size + 1) % 7.0))


def put(name, seed, view, x, y, params, rep, want):
    store[f"{name}/sim"] = np.asarray(rep.y_out)
    if want is not None:
        store[f"{name}/naive"] = np.asarray(want)
    p = dict(params)
    p.update(seed=seed, rows=view.rows, cols=view.cols, ld=view.ld, xl=len(x), yl=len(y),
             tag=view.precision.tag, flops=int(rep.flops), scal_invocations=int(rep.scal_invocations),
             sum_A=checksum(view.data), sum_x=checksum(x), sum_y=checksum(y))
    meta[name] = p


def main():
    cfg = KernelConfig(32, 4, coop_tbs=2)
    for tag in "sdcz":
        for trans in "ntc":
            for m, n in [(1, 1), (7, 5), (32, 32), (65, 33), (100, 300)]:
                xl, yl = (n, m) if trans == "n" else (m, n)
                seed, a, x, y = case_inputs(m, n, xl, yl, tag)
                rep = blockmv.gemv(trans, 0.7, a, x, -0.3, y, cfg)
                want = blockmv.naive_gemv(trans, 0.7, a, x, -0.3, y)
                put(f"gemv_{tag}{trans}_{m}x{n}", seed, a, x, y,
                    dict(op="gemv", trans=trans, alpha=0.7, beta=-0.3, nb=32, coop=2), rep, want)
    cfg = KernelConfig(32, 2, coop_tbs=2)
    for tag in "sdcz":
        for uplo in "lu":
            for d in (1, 5, 32, 33, 100, 257):
                for herm in ([True, False] if tag in "cz" else [False]):
                    seed, a, x, y = case_inputs(d, d, d, d, tag)
                    hv = HermitianView(base=a, uplo=uplo)
                    rep = blockmv.symv_hemv(uplo, 1.1, hv, x, -0.2, y, cfg, hermitian=herm)
                    want = blockmv.naive_symv_hemv(1.1, hv, x, -0.2, y, hermitian=herm)
                    put(f"symv_{tag}{uplo}{'h' if herm else 's'}_{d}", seed, a, x, y,
                        dict(op="symv", uplo=uplo, hermitian=herm, alpha=1.1, beta=-0.2, nb=32, coop=2),
                        rep, want)
    # offsets (test_offset.py:39-62, 124-145 shapes)
    cfg = KernelConfig(32, 2, coop_tbs=2)
    rng = np.random.default_rng(41)
    for tag in "sdcz":
        for trans in "ntc":
            for k in range(3):
                pm, pn = int(rng.integers(40, 200)), int(rng.integers(40, 200))
                sm, sn = int(rng.integers(1, pm)), int(rng.integers(1, pn))
                ro, co = int(rng.integers(0, pm - sm + 1)), int(rng.integers(0, pn - sn + 1))
                xl, yl = (sn, sm) if trans == "n" else (sm, sn)
                seed, parent, x, y = case_inputs(pm, pn, xl, yl, tag)
                req = blockmv.OffsetRequest(parent=parent, row_off=ro, col_off=co, sub_m=sm, sub_n=sn)
                rep = blockmv.gemv_offset(trans, 0.9, req, x, -1.2, y, cfg)
                want = blockmv.naive_gemv(trans, 0.9, parent.submatrix(ro, co, sm, sn), x, -1.2, y)
                put(f"gemvoff_{tag}{trans}_{k}", seed, parent, x, y,
                    dict(op="gemv_offset", trans=trans, alpha=0.9, beta=-1.2, nb=32, coop=2,
                         row_off=ro, col_off=co, sub_m=sm, sub_n=sn), rep, want)
    rng = np.random.default_rng(46)
    for tag in "sdcz":
        for uplo in "lu":
            for k in range(3):
                pd = int(rng.integers(64, 300))
                sd = int(rng.integers(1, pd))
                off = int(rng.integers(0, pd - sd + 1))
                seed, pmat, x, y = case_inputs(pd, pd, sd, sd, tag)
                parent = HermitianView(base=pmat, uplo=uplo)
                rep = blockmv.symv_hemv_offset(uplo, 0.8, parent, off, sd, x, -0.4, y, KernelConfig(32, 2))
                sub_hv = HermitianView(base=pmat.submatrix(off, off, sd, sd), uplo=uplo)
                want = blockmv.naive_symv_hemv(0.8, sub_hv, x, -0.4, y)
                put(f"symvoff_{tag}{uplo}_{k}", seed, pmat, x, y,
                    dict(op="symv_offset", uplo=uplo, hermitian=tag in "cz", alpha=0.8, beta=-0.4, nb=32,
                         coop=1, offset=off, sub_d=sd), rep, want)
    # mgpu (test_multidevice.py:75-146)
    for G in (1, 2, 4, 8):
        for trans, tag in (("n", "d"), ("t", "d"), ("c", "z")):
            for d in (64, 100, 256):
                seed, a, x, y = case_inputs(d, d, d, d, tag)
                merged, _ = blockmv.gemv_mgpu(trans, 1.2, blockmv.distribute(a, 32, G), x, -0.5, y,
                                              KernelConfig(32, 2))
                want = blockmv.naive_gemv(trans, 1.2, a, x, -0.5, y)
                put(f"gemvmgpu_{tag}{trans}_G{G}_{d}", seed, a, x, y,
                    dict(op="gemv_mgpu", trans=trans, alpha=1.2, beta=-0.5, nb=32, coop=1, G=G), merged, want)
    for G in (1, 2, 3, 8):
        for tag, uplo in (("d", "l"), ("d", "u"), ("c", "l"), ("z", "u")):
            for d in (64, 100, 256):
                seed, a, x, y = case_inputs(d, d, d, d, tag)
                hv = HermitianView(base=a, uplo=uplo)
                merged, _ = blockmv.symv_hemv_mgpu(uplo, 0.9, blockmv.distribute(a, 32, G), x, 0.7, y,
                                                   KernelConfig(32, 2))
                want = blockmv.naive_symv_hemv(0.9, hv, x, 0.7, y)
                put(f"symvmgpu_{tag}{uplo}_G{G}_{d}", seed, a, x, y,
                    dict(op="symv_mgpu", uplo=uplo, hermitian=tag in "cz", alpha=0.9, beta=0.7, nb=32, coop=1,
                         G=G), merged, want)
    # BASELINE config 1: DGEMV N=4096, alpha=1, beta=0, cli.py recipe (A -> x -> y, seed 0)
    rng = np.random.default_rng(0)
    prec = precision("d")
    n = 4096
    a = make_padded_view(n, n, prec, pad_to=32)
    a.array()[:, :] = rng.uniform(-1, 1, size=(n, n)).astype(np.float64)
    x = rng.uniform(-1, 1, size=n).astype(np.float64)
    y = rng.uniform(-1, 1, size=n).astype(np.float64)
    rep = blockmv.gemv("n", 1.0, a, x, 0.0, y, KernelConfig(64, 4, 1))
    want = blockmv.naive_gemv("n", 1.0, a, x, 0.0, y)
    store["cfg1_dgemv_4096/sim"] = np.asarray(rep.y_out)
    store["cfg1_dgemv_4096/naive"] = np.asarray(want)
    meta["cfg1_dgemv_4096"] = dict(op="gemv_cfg1", trans="n", alpha=1.0, beta=0.0, n=n, seed=0,
                                   recipe="cli.py:52-57,100-125: A(n,n) -> x(n) -> y(n), U(-1,1)",
                                   flops=int(rep.flops), scal_invocations=int(rep.scal_invocations))
    store["__meta__"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT}: {len(meta)} cases, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
