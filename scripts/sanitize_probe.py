#!/usr/bin/env python
"""One small call of every kernel family (and form) for compute-sanitizer:

    compute-sanitizer --tool memcheck python scripts/sanitize_probe.py
    compute-sanitizer --tool racecheck python scripts/sanitize_probe.py
    compute-sanitizer --tool synccheck python scripts/sanitize_probe.py

Ragged sizes and a misaligned submatrix start so predicated edges run.
Exits non-zero if any result is non-finite."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1410_1726_b200 as kb  # noqa: E402
from paper_1410_1726_b200 import _lib  # noqa: E402

lib = _lib.load()
torch.manual_seed(0)
bad = 0


def mat(tag, m, n, ld, ro):
    p = kb.precision(tag)
    buf = torch.empty(ld * (n + 1), dtype=p.torch_dtype, device="cuda")
    (torch.view_as_real(buf) if p.is_complex else buf).uniform_(-1, 1)
    return kb.MatrixView(buf, ro + m, n + 1, ld, p).submatrix(ro, 1, m, n)


def vec(tag, n):
    p = kb.precision(tag)
    v = torch.empty(n, dtype=p.torch_dtype, device="cuda")
    (torch.view_as_real(v) if p.is_complex else v).uniform_(-1, 1)
    return v


def ok(name, t):
    global bad
    torch.cuda.synchronize()
    if not torch.isfinite(t).all():
        print("non-finite:", name)
        bad += 1


forms = [
    ("default", lambda: None),
    ("split-slots", lambda: (_lib.set_gemv_split(1), lib.kblas_set_gemv_cluster(0))),
    ("split-cluster", lambda: (_lib.set_gemv_split(1), lib.kblas_set_gemv_cluster(1))),
    ("stacked", lambda: (_lib.set_gemv_split(0), lib.kblas_set_gemv_cluster(-1))),
    ("t-streamk", lambda: (_lib.set_gemv_split(-1), lib.kblas_set_gemv_tc(0, 0))),
    ("t-colown", lambda: lib.kblas_set_gemv_tc(1, 0)),
    ("rowown0", lambda: (lib.kblas_set_gemv_tc(-1, 0), lib.kblas_set_gemv_split(3), lib.kblas_set_gemv_rowown(0))),
    ("rowown2", lambda: lib.kblas_set_gemv_rowown(2)),
    ("rowown7", lambda: lib.kblas_set_gemv_rowown(7)),
]
for tag in "sdcz":
    for m, n, ld, ro in ((333, 517, 352, 3), (1025, 300, 1056, 0), (4100, 77, 4128, 5)):
        A = mat(tag, m, n, ld, ro)
        for fname, setf in forms:
            setf()
            for trans in "ntc":
                xl, yl = (n, m) if trans == "n" else (m, n)
                r = kb.gemv(trans, 0.5, A, vec(tag, xl), 0.25, vec(tag, yl)).y_out
                ok(f"gemv {tag} {trans} {fname}", r)
        _lib.set_gemv_split(-1)
        lib.kblas_set_gemv_cluster(-1)
        lib.kblas_set_gemv_tc(-1, 0)
        lib.kblas_set_gemv_rowown(-1)
    d, ld, ro = 700, 736, 5
    A = mat(tag, d + 1, d + 1, ld, ro).submatrix(0, 0, d, d)
    herm = tag in "cz"
    for uplo in "lu":
        for narrow in (0, 1 << 30):
            _lib.set_symv_narrow(narrow)
            r = kb.symv_hemv(uplo, 0.5, kb.HermitianView(A, uplo), vec(tag, d), 0.25, vec(tag, d),
                             hermitian=herm).y_out
            ok(f"symv {tag} {uplo} narrow={narrow}", r)
        _lib.set_symv_narrow(2048)
        prev = _lib.set_tma(1)
        r = kb.symv_hemv(uplo, 0.5, kb.HermitianView(A, uplo), vec(tag, d), 0.25, vec(tag, d), hermitian=herm).y_out
        ok(f"symv-tma {tag} {uplo}", r)
        _lib.set_tma(prev)
    # 128-wide tiles (the 128-row epilogue): the 2-CTA/SM variant off, on
    # the single-GPU path (uniform tiles) and on mgpu panels with nb = 128
    prev_mid = lib.kblas_set_symv_mid(0)
    for uplo in "lu":
        for beta in (0.0, 0.25):
            r = kb.symv_hemv(uplo, 0.5, kb.HermitianView(A, uplo), vec(tag, d), beta, vec(tag, d),
                             hermitian=herm).y_out
            ok(f"symv wide {tag} {uplo} beta={beta}", r)
    lib.kblas_set_symv_mid(prev_mid)
    dist = kb.distribute(kb.view_of(torch.rand(1000, 1000, device="cuda", dtype=kb.precision(tag).torch_dtype).T),
                         128, 3)
    r = kb.symv_hemv_mgpu("l", 1.0, dist, vec(tag, 1000), 0.5, vec(tag, 1000), kb.KernelConfig(128, 2),
                          hermitian=herm)[0].y_out
    ok(f"symv mgpu nb=128 {tag}", r)
    dist = kb.distribute(kb.view_of(torch.rand(600, 600, device="cuda", dtype=kb.precision(tag).torch_dtype).T),
                         64, 3)
    r = kb.symv_hemv_mgpu("l", 1.0, dist, vec(tag, 600), 0.5, vec(tag, 600), kb.KernelConfig(64, 2),
                          hermitian=herm)[0].y_out
    ok(f"symv mgpu {tag}", r)
    r = kb.gemv_mgpu("n", 1.0, dist, vec(tag, 600), 0.5, vec(tag, 600))[0].y_out
    ok(f"gemv mgpu {tag}", r)
# split SYMV schedule (tail grid of small CTAs, last CTA waits for the
# first grid): device vectors and a page-locked x (tail grid waits at start)
for tag, d in (("d", 16384), ("c", 16384)):
    p = kb.precision(tag)
    A = torch.empty(d, d, dtype=p.torch_dtype, device="cuda")
    (torch.view_as_real(A) if p.is_complex else A).uniform_(-1, 1)
    hv = kb.HermitianView(kb.view_of(A.T), "l")
    r = kb.symv_hemv("l", 1.0, hv, vec(tag, d), 0.5, vec(tag, d)).y_out
    ok(f"symv split {tag} plan={_lib.last_plan().split()[-1]}", r)
    hx = torch.empty(d, dtype=p.torch_dtype, pin_memory=True)
    hx.copy_(vec(tag, d))
    r = kb.symv_hemv("l", 1.0, hv, hx.numpy(), 0.0, torch.zeros(d, dtype=p.torch_dtype).numpy()).y_out
    if not (r == r).all():
        print("non-finite: symv split hostvec", tag)
        bad += 1
    del A
# host-vector path: page-locked x / y (copy-in grid + PDL-launched main
# kernel with the prefetch-before-wait prologue), misaligned pinned views,
# pageable vectors, and queued calls
import numpy as np  # noqa: E402


def pinned(tag, n, shift=0):
    p = kb.precision(tag)
    t = torch.empty(n + shift, dtype=p.torch_dtype, pin_memory=True)
    (torch.view_as_real(t) if p.is_complex else t).uniform_(-1, 1)
    return t.numpy()[shift:]


def ok_np(name, a):
    global bad
    if not np.isfinite(a).all():
        print("non-finite:", name)
        bad += 1


for tag in "sdcz":
    herm = tag in "cz"
    for m, n, ld, ro in ((333, 517, 352, 3), (4100, 77, 4128, 5), (2048, 2048, 2048, 0)):
        A = mat(tag, m, n, ld, ro)
        for trans in "ntc":
            xl, yl = (n, m) if trans == "n" else (m, n)
            for shift in (0, 1):
                for beta in (0.0, 0.25):
                    r = kb.gemv(trans, 0.5, A, pinned(tag, xl, shift), beta, pinned(tag, yl, shift)).y_out
                    ok_np(f"hostvec gemv {tag} {trans} shift={shift} beta={beta}", r)
            r = kb.gemv(trans, 0.5, A, pinned(tag, xl).copy(), 0.25, pinned(tag, yl).copy()).y_out
            ok_np(f"hostvec gemv pageable {tag} {trans}", r)
    d, ld, ro = 700, 736, 5
    A = mat(tag, d + 1, d + 1, ld, ro).submatrix(0, 0, d, d)
    for uplo in "lu":
        for beta in (0.0, 0.25):
            r = kb.symv_hemv(uplo, 0.5, kb.HermitianView(A, uplo), pinned(tag, d, 1), beta, pinned(tag, d),
                             hermitian=herm).y_out
            ok_np(f"hostvec symv {tag} {uplo} beta={beta}", r)
    q = kb.CommandQueue()
    hs = [kb.gemv_async("n", 1.0, A, pinned(tag, d), 0.0, np.zeros(d, dtype=kb.precision(tag).dtype), queue=q)
          for _ in range(4)]
    q.synchronize()
    for h in hs:
        ok_np(f"hostvec queued {tag}", h.result().y_out)
print("sanitize probe done, bad =", bad)
sys.exit(1 if bad else 0)
