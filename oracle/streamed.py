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
        _lib = lib
    return _lib


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
