"""ctypes wrapper of oracle/streamed.c (test infrastructure only)."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "streamed.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        vp = ctypes.c_void_p
        lib.oracle_gemv.argtypes = [ctypes.c_char, ctypes.c_char, ctypes.c_int, ctypes.c_int, dp, vp,
                                    ctypes.c_longlong, vp, dp, vp, dp, ctypes.c_int]
        lib.oracle_gemv.restype = ctypes.c_int
        lib.oracle_symv.argtypes = [ctypes.c_char, ctypes.c_char, ctypes.c_int, ctypes.c_int, dp, vp,
                                    ctypes.c_longlong, vp, dp, vp, dp, ctypes.c_int]
        lib.oracle_symv.restype = ctypes.c_int
        lib.oracle_symv_norm_inf.argtypes = [ctypes.c_char, ctypes.c_char, ctypes.c_int, ctypes.c_int, vp,
                                             ctypes.c_longlong]
        lib.oracle_symv_norm_inf.restype = ctypes.c_double
        lib.oracle_max_threads.restype = ctypes.c_int
        u64, ll = ctypes.c_ulonglong, ctypes.c_longlong
        lib.oracle_gemv_gen.argtypes = [ctypes.c_char, ctypes.c_char, ctypes.c_int, ctypes.c_int, u64, ll, ll, ll,
                                        dp, vp, dp, vp, dp, dp, ctypes.c_int]
        lib.oracle_gemv_gen.restype = ctypes.c_int
        lib.oracle_symv_gen.argtypes = [ctypes.c_char, ctypes.c_char, ctypes.c_int, ctypes.c_int, u64, ll, ll,
                                        dp, vp, dp, vp, dp, dp, ctypes.c_int]
        lib.oracle_symv_gen.restype = ctypes.c_int
        lib.oracle_gen_fill.argtypes = [ctypes.c_char, ctypes.c_int, ctypes.c_int, u64, ll, ll, ll, vp, ll,
                                        ctypes.c_int]
        lib.oracle_gen_fill.restype = ctypes.c_int
        lib.oracle_gen_fill_tri.argtypes = [ctypes.c_char, ctypes.c_char, ctypes.c_int, u64, ll, vp, ll, ctypes.c_int]
        lib.oracle_gen_fill_tri.restype = ctypes.c_int
        _lib = lib
    return _lib


DTYPES = {"s": np.float32, "d": np.float64, "c": np.complex64, "z": np.complex128}
TAG = {np.dtype(np.float32): "s", np.dtype(np.float64): "d", np.dtype(np.complex64): "c",
       np.dtype(np.complex128): "z"}


def _wide2(v):
    v = complex(v)
    return (ctypes.c_double * 2)(v.real, v.imag)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _flat(a2d):
    """(buffer, lda) of a column-major 2-D view (unit row stride)."""
    a2d = np.asarray(a2d)
    item = a2d.itemsize
    if a2d.shape[0] <= 1 and a2d.shape[1] <= 1:
        return np.ascontiguousarray(a2d), max(1, a2d.shape[0])
    if a2d.strides[0] != item:
        a2d = np.asfortranarray(a2d)
    lda = a2d.strides[1] // item if a2d.shape[1] > 1 else a2d.shape[0]
    return a2d, max(lda, 1)


def _out(tag, wide, dtype):
    w = wide.view(np.complex128)
    return (w if tag in "cz" else w.real).astype(dtype)


def gemv(trans, alpha, a2d, x, beta, y, nthreads: int = 0, wide_out: bool = False):
    """naive_gemv restated (reference.py:39-50)."""
    a, lda = _flat(a2d)
    tag = TAG[a.dtype]
    trans = trans.lower()
    if trans == "c" and tag in "sd":
        trans = "t"
    m, n = a.shape
    x = np.ascontiguousarray(x, dtype=a.dtype)
    y = np.ascontiguousarray(y, dtype=a.dtype)
    ylen = m if trans == "n" else n
    out = np.zeros(2 * ylen, dtype=np.float64)
    rc = load().oracle_gemv(tag.encode(), trans.encode(), m, n, _wide2(alpha), _ptr(a), lda, _ptr(x),
                            _wide2(beta), _ptr(y), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                            nthreads)
    assert rc == 0
    return out.view(np.complex128) if wide_out else _out(tag, out, a.dtype)


def symv(uplo, alpha, a2d, x, beta, y, hermitian=None, nthreads: int = 0, wide_out: bool = False):
    """naive_symv_hemv restated (reference.py:53-59), triangle streamed."""
    a, lda = _flat(a2d)
    tag = TAG[a.dtype]
    if hermitian is None:
        hermitian = tag in "cz"
    n = a.shape[0]
    x = np.ascontiguousarray(x, dtype=a.dtype)
    y = np.ascontiguousarray(y, dtype=a.dtype)
    out = np.zeros(2 * n, dtype=np.float64)
    rc = load().oracle_symv(tag.encode(), uplo.lower().encode(), int(bool(hermitian)), n, _wide2(alpha),
                            _ptr(a), lda, _ptr(x), _wide2(beta), _ptr(y),
                            out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), nthreads)
    assert rc == 0
    return out.view(np.complex128) if wide_out else _out(tag, out, a.dtype)


def symv_norm_inf(uplo, a2d, hermitian=None) -> float:
    a, lda = _flat(a2d)
    tag = TAG[a.dtype]
    if hermitian is None:
        hermitian = tag in "cz"
    return float(load().oracle_symv_norm_inf(tag.encode(), uplo.lower().encode(), int(bool(hermitian)),
                                             a.shape[0], _ptr(a), lda))


def max_threads() -> int:
    return int(load().oracle_max_threads())


# ------------------------------------------------ generated operands
# The operand is regenerated inside the C loops from a counter-based
# generator (streamed.c header; oracle/gen.py restates it for the device),
# so no host copy of a 28-160 GB matrix is needed.
KEY_LIMIT = 1 << 36


def _check_keys(tag, gen_ld, rows, cols):
    kmax = (cols * gen_ld + rows) * (2 if tag in "cz" else 1)
    if kmax >= KEY_LIMIT:
        raise ValueError("generated operand too large for the 36-bit key space")


def gemv_gen(tag, trans, m, n, seed, gen_ld, ro, co, alpha, x, beta, y, nthreads: int = 0,
             wide_out: bool = False):
    """naive_gemv (reference.py:39-50) on the m x n operand generated with
    (seed, gen_ld) at offset (ro, co).  Returns (y_out, ||op(A)||_inf)."""
    dt = DTYPES[tag]
    trans = trans.lower()
    if trans == "c" and tag in "sd":
        trans = "t"
    _check_keys(tag, gen_ld, ro + m, co + n)
    x = np.ascontiguousarray(x, dtype=dt)
    y = np.ascontiguousarray(y, dtype=dt)
    ylen = m if trans == "n" else n
    out = np.zeros(2 * ylen, dtype=np.float64)
    norm = ctypes.c_double(0.0)
    rc = load().oracle_gemv_gen(tag.encode(), trans.encode(), m, n, seed, gen_ld, ro, co, _wide2(alpha), _ptr(x),
                                _wide2(beta), _ptr(y), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                ctypes.byref(norm), nthreads)
    assert rc == 0
    return (out.view(np.complex128) if wide_out else _out(tag, out, dt)), norm.value


def symv_gen(tag, uplo, n, seed, gen_ld, off, alpha, x, beta, y, hermitian=None, nthreads: int = 0,
             wide_out: bool = False):
    """naive_symv_hemv (reference.py:53-59) on the diagonal n x n block at
    (off, off) of the generated operand.  Returns (y_out, ||A_dense||_inf)."""
    dt = DTYPES[tag]
    if hermitian is None:
        hermitian = tag in "cz"
    _check_keys(tag, gen_ld, off + n, off + n)
    x = np.ascontiguousarray(x, dtype=dt)
    y = np.ascontiguousarray(y, dtype=dt)
    out = np.zeros(2 * n, dtype=np.float64)
    norm = ctypes.c_double(0.0)
    rc = load().oracle_symv_gen(tag.encode(), uplo.lower().encode(), int(bool(hermitian)), n, seed, gen_ld, off,
                                _wide2(alpha), _ptr(x), _wide2(beta), _ptr(y),
                                out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(norm), nthreads)
    assert rc == 0
    return (out.view(np.complex128) if wide_out else _out(tag, out, dt)), norm.value


def gen_fill(tag, m, n, seed, gen_ld, ro=0, co=0, nthreads: int = 0):
    """The generated m x n operand at (ro, co), materialised (Fortran order)."""
    _check_keys(tag, gen_ld, ro + m, co + n)
    out = np.zeros((n, m), dtype=DTYPES[tag])  # row j = column j
    rc = load().oracle_gen_fill(tag.encode(), m, n, seed, gen_ld, ro, co, _ptr(out), m, nthreads)
    assert rc == 0
    return out.T
