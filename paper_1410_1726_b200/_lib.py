"""ctypes binding of the C ABI declared in include/kblas_b200.h.

The shared library is the only compute path: if it is missing or cannot be
loaded this module raises, it never falls back to a CPU implementation.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_char, c_double, c_float, c_int, c_size_t, c_ulonglong, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
# KBLAS_LIB: load another build of the library (same-box A/B runs of two
# builds, scripts/*_ab.sh); the default is the in-tree build
LIB_PATH = os.environ.get("KBLAS_LIB") or os.path.join(HERE, "libkblas_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "kblas_b200.h")


class c_complex64(ctypes.Structure):
    _fields_ = [("re", c_float), ("im", c_float)]


class c_complex128(ctypes.Structure):
    _fields_ = [("re", c_double), ("im", c_double)]


SCALAR_CTYPE = {"s": c_float, "d": c_double, "c": c_complex64, "z": c_complex128}


def scalar(tag: str, value):
    """Host scalar of precision `tag` for a by-value C argument."""
    ct = SCALAR_CTYPE[tag]
    if tag in "cz":
        v = complex(value)
        return ct(v.real, v.imag)
    if isinstance(value, complex):
        if value.imag != 0:
            raise ValueError(f"complex scalar {value!r} for real precision {tag!r}")
        value = value.real
    return ct(float(value))


_lock = threading.Lock()
_lib = None

_GEMV = ["trans", "m", "n", "alpha", "A", "lda", "x", "incx", "beta", "y", "incy"]
_SYMV = ["uplo", "n", "alpha", "A", "lda", "x", "incx", "beta", "y", "incy"]
SYMV_NAMES = {"s": ["ssymv"], "d": ["dsymv"], "c": ["chemv", "csymv"], "z": ["zhemv", "zsymv"]}


def _argtypes(kind, tag, extra=()):
    s = SCALAR_CTYPE[tag]
    if kind == "gemv":
        base = [c_char, c_int, c_int, s, c_void_p, c_int, c_void_p, c_int, s, c_void_p, c_int]
    else:
        base = [c_char, c_int, s, c_void_p, c_int, c_void_p, c_int, s, c_void_p, c_int]
    return base + list(extra)


def _mgpu_argtypes(kind, tag):
    s = SCALAR_CTYPE[tag]
    pp = POINTER(c_void_p)
    if kind == "gemv":
        return [c_char, c_int, c_int, s, pp, c_int, pp, c_int, s, pp, c_int, c_int, c_int, POINTER(c_int)]
    return [c_char, c_int, s, pp, c_int, pp, c_int, s, pp, c_int, c_int, c_int, POINTER(c_int)]


def load():
    """Load (once) and return the library with all prototypes set."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1410_1726_b200._build` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for tag in "sdcz":
            for suffix, extra in (
                ("", ()),
                ("_async", (c_void_p,)),
                ("_offset", (c_int, c_int)),
                ("_offset_async", (c_int, c_int, c_void_p)),
            ):
                f = getattr(lib, f"kblas_{tag}gemv{suffix}")
                f.argtypes = _argtypes("gemv", tag, extra)
                f.restype = c_int
            getattr(lib, f"kblas_{tag}gemv_mgpu").argtypes = _mgpu_argtypes("gemv", tag)
            getattr(lib, f"kblas_{tag}gemv_mgpu").restype = c_int
            getattr(lib, f"kblas_{tag}gemv_mgpu_async").argtypes = _mgpu_argtypes("gemv", tag) + [POINTER(c_void_p)]
            getattr(lib, f"kblas_{tag}gemv_mgpu_async").restype = c_int
            for name in SYMV_NAMES[tag]:
                for suffix, extra in (
                    ("", ()),
                    ("_async", (c_void_p,)),
                    ("_offset", (c_int,)),
                    ("_offset_async", (c_int, c_void_p)),
                ):
                    f = getattr(lib, f"kblas_{name}{suffix}")
                    f.argtypes = _argtypes("symv", tag, extra)
                    f.restype = c_int
                getattr(lib, f"kblas_{name}_mgpu").argtypes = _mgpu_argtypes("symv", tag)
                getattr(lib, f"kblas_{name}_mgpu").restype = c_int
                getattr(lib, f"kblas_{name}_mgpu_async").argtypes = (_mgpu_argtypes("symv", tag)
                                                                     + [POINTER(c_void_p)])
                getattr(lib, f"kblas_{name}_mgpu_async").restype = c_int
        lib.kblas_mv_mgpu_combine_async.argtypes = [c_char, ctypes.c_longlong, c_int, POINTER(c_void_p), c_void_p,
                                                     c_void_p, c_void_p]
        lib.kblas_mv_mgpu_combine_async.restype = c_int
        lib.kblas_mv_mgpu_partial_async.argtypes = [
            c_char, c_char, c_char, c_int, c_int, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
            c_int, c_int, c_int, c_int, c_void_p,
        ]
        lib.kblas_mv_mgpu_partial_async.restype = c_int
        lib.kblas_ipc_get_handle.argtypes = [c_void_p, c_void_p]
        lib.kblas_ipc_open_handle.argtypes = [c_void_p, POINTER(c_void_p)]
        lib.kblas_ipc_close.argtypes = [c_void_p]
        lib.kblas_p2p_signal_async.argtypes = [c_void_p, c_ulonglong, c_void_p]
        lib.kblas_p2p_wait_async.argtypes = [c_void_p, c_ulonglong, c_void_p]
        lib.kblas_p2p_combine_async.argtypes = [c_char, c_int, c_void_p, ctypes.c_longlong, c_void_p, c_ulonglong,
                                                c_void_p, c_void_p, ctypes.c_longlong, c_void_p, c_void_p, c_void_p]
        lib.kblas_mv_mgpu_partial_p2p_async.argtypes = [
            c_char, c_char, c_char, c_int, c_int, c_void_p, c_void_p, c_int, c_void_p, c_int, c_int, c_int, c_int,
            c_void_p, ctypes.c_longlong, c_void_p, c_void_p, c_void_p, c_ulonglong, c_void_p, c_void_p, c_void_p,
            c_void_p]
        lib.kblas_mv_mgpu_partial_p2p_async.restype = c_int
        for name in ("kblas_ipc_get_handle", "kblas_ipc_open_handle", "kblas_ipc_close", "kblas_p2p_signal_async",
                     "kblas_p2p_wait_async", "kblas_p2p_combine_async"):
            getattr(lib, name).restype = c_int
        lib.kblas_mv_hostvec.argtypes = [
            c_char, c_char, c_char, c_int, c_int, c_int, c_void_p, c_void_p, c_int, c_int, c_int,
            c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
        ]
        lib.kblas_mv_hostvec.restype = c_int
        lib.kblas_mv_hostvec_async.argtypes = [
            c_char, c_char, c_char, c_int, c_int, c_int, c_void_p, c_void_p, c_int, c_int, c_int,
            c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
        ]
        lib.kblas_mv_hostvec_async.restype = c_int
        lib.kblas_stream_sync.argtypes = [c_void_p]
        lib.kblas_stream_sync.restype = c_int
        lib.kblas_stream_order.argtypes = [c_void_p, c_void_p]
        lib.kblas_stream_order.restype = c_int
        lib.kblas_mgpu_local_cols.argtypes = [c_int, c_int, c_int, c_int]
        lib.kblas_mgpu_local_cols.restype = c_int
        lib.kblas_malloc_mgpu_1d.argtypes = [c_int, c_int, c_size_t, POINTER(c_void_p), POINTER(c_int), c_int,
                                             c_int, POINTER(c_int)]
        lib.kblas_malloc_mgpu_1d.restype = c_int
        lib.kblas_free_mgpu.argtypes = [POINTER(c_void_p), c_int, POINTER(c_int)]
        lib.kblas_free_mgpu.restype = c_int
        lib.kblas_mgpu_block_size.argtypes = [c_char, c_char]
        lib.kblas_mgpu_block_size.restype = c_int
        lib.kblas_mgpu_local_ld.argtypes = [c_int]
        lib.kblas_mgpu_local_ld.restype = c_int
        for name in ("kblas_setmatrix_mgpu_1d", "kblas_getmatrix_mgpu_1d"):
            getattr(lib, name).restype = c_int
        lib.kblas_setmatrix_mgpu_1d.argtypes = [
            c_int, c_int, c_size_t, c_void_p, c_int, POINTER(c_void_p), c_int, c_int, c_int, POINTER(c_int)]
        lib.kblas_getmatrix_mgpu_1d.argtypes = [
            c_int, c_int, c_size_t, POINTER(c_void_p), c_int, c_void_p, c_int, c_int, c_int, POINTER(c_int)]
        for name in ("kblas_setmatrix_async", "kblas_getmatrix_async"):
            getattr(lib, name).argtypes = [c_int, c_int, c_size_t, c_void_p, c_int, c_void_p, c_int, c_void_p]
            getattr(lib, name).restype = c_int
        lib.kblas_clear_cache.argtypes = []
        lib.kblas_clear_cache.restype = c_int
        lib.kblas_launch_count.restype = c_ulonglong
        lib.kblas_launch_count.argtypes = []
        lib.kblas_timing_enable.argtypes = [c_int]
        lib.kblas_timing_enable.restype = c_int
        lib.kblas_timing_read.argtypes = [POINTER(c_double), POINTER(c_int)]
        lib.kblas_timing_read.restype = c_int
        lib.kblas_set_symv_variant.argtypes = [c_int]
        lib.kblas_set_symv_variant.restype = c_int
        lib.kblas_set_tma.argtypes = [c_int]
        lib.kblas_set_tma.restype = c_int
        lib.kblas_set_gemv_cluster.argtypes = [c_int]
        lib.kblas_set_gemv_cluster.restype = c_int
        lib.kblas_set_gemv_split_waves.argtypes = [c_int]
        lib.kblas_set_gemv_split_waves.restype = c_int
        lib.kblas_set_gemv_tc.argtypes = [c_int, ctypes.c_longlong]
        lib.kblas_set_gemv_tc.restype = c_int
        lib.kblas_set_gemv_variant.argtypes = [c_int]
        lib.kblas_set_gemv_variant.restype = c_int
        lib.kblas_set_gemv_rowown.argtypes = [c_int]
        lib.kblas_set_gemv_rowown.restype = c_int
        lib.kblas_set_gemv_split.argtypes = [c_int]
        lib.kblas_set_gemv_split.restype = c_int
        lib.kblas_set_symv_mid.argtypes = [c_int]
        lib.kblas_set_symv_mid.restype = c_int
        lib.kblas_set_symv_window.argtypes = [c_int]
        lib.kblas_set_symv_window.restype = c_int
        lib.kblas_set_symv_segment.argtypes = [c_int]
        lib.kblas_set_symv_segment.restype = c_int
        lib.kblas_set_symv_trace.argtypes = [c_void_p]
        lib.kblas_set_symv_trace.restype = c_int
        lib.kblas_set_symv_narrow.argtypes = [c_int]
        lib.kblas_set_symv_narrow.restype = c_int
        LL = ctypes.c_longlong
        lib.kblas_tune_set.argtypes = [c_char, c_char, LL, LL, c_int, c_int, c_int]
        lib.kblas_tune_set.restype = c_int
        lib.kblas_tune_clear.argtypes = []
        lib.kblas_tune_clear.restype = c_int
        lib.kblas_tune_defaults.argtypes = []
        lib.kblas_tune_defaults.restype = c_int
        lib.kblas_tune_count.argtypes = []
        lib.kblas_tune_count.restype = c_int
        lib.kblas_tune_get.argtypes = [c_int, ctypes.c_char_p, ctypes.c_char_p, POINTER(LL), POINTER(LL),
                                       POINTER(c_int), POINTER(c_int), POINTER(c_int)]
        lib.kblas_tune_get.restype = c_int
        lib.kblas_last_plan.restype = ctypes.c_char_p
        lib.kblas_last_plan.argtypes = []
        lib.kblas_version.restype = ctypes.c_char_p
        lib.kblas_version.argtypes = []
        _lib = lib
        path = os.environ.get("KBLAS_TUNING_FILE")
        if path:
            _load_tuning(lib, path)
        return lib


def _load_tuning(lib, path: str):
    """Install the tuning table saved at `path` (paper_1410_1726_b200.tuner
    .save format); a bad file raises rather than running untuned silently."""
    import json

    with open(path) as fh:
        doc = json.load(fh)
    if doc.get("format") != "kblas-b200-tuning/1":
        raise ValueError(f"{path}: not a kblas-b200 tuning table")
    for e in doc["entries"]:
        rc = lib.kblas_tune_set(e["prec"].encode(), e["op"].encode(), int(e["n_lo"]), int(e["n_hi"]),
                                int(e["shape"]), int(e.get("form", -1)), int(e.get("waves", 0)))
        check(rc, f"{path}: kblas_tune_set", ["prec", "op", "n_lo", "n_hi", "shape", "form", "waves"])


def header_symbols() -> list[str]:
    """Every kblas_* function declared in include/kblas_b200.h."""
    import re

    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kblas_\w+)\s*\(", text)))


class KblasError(RuntimeError):
    pass


def check(rc: int, what: str, argnames=None):
    if rc == 0:
        return
    if rc < 0:
        k = -rc
        name = argnames[k - 1] if argnames and 0 < k <= len(argnames) else f"#{k}"
        raise ValueError(f"{what}: invalid argument {k} ({name})")
    raise KblasError(f"{what}: CUDA error {rc}")


def launch_count() -> int:
    return int(load().kblas_launch_count())


def last_plan() -> str:
    return load().kblas_last_plan().decode()


def set_tma(mode) -> int:
    """SYMV/HEMV kernel: True/1 TMA-fed pipeline, False/0 register-load
    kernel, -1 tuned per-precision default.  Returns the previous mode."""
    m = -1 if mode == -1 else (1 if mode else 0)
    return int(load().kblas_set_tma(m))


def set_gemv_split(mode) -> int:
    """GEMV-N form: True/1 split form always, False/0 never, -1 automatic.
    Returns the previous mode."""
    m = -1 if mode == -1 else (1 if mode else 0)
    return int(load().kblas_set_gemv_split(m))


def set_symv_window(items: int) -> int:
    """Register SYMV/HEMV kernel: row chunks per CTA barrier window (1, 2
    or 4).  Returns the previous value."""
    return int(load().kblas_set_symv_window(int(items)))


def set_symv_segment(items: int) -> int:
    """SYMV/HEMV schedule: segments of `items` row chunks round robin over
    the CTAs (<= 0: contiguous stream-K).  Returns the previous value."""
    return int(load().kblas_set_symv_segment(int(items)))


def set_symv_narrow(max_order: int) -> int:
    """Register SYMV/HEMV: narrow tiles up to this order.  Returns the
    previous threshold."""
    return int(load().kblas_set_symv_narrow(int(max_order)))


def timing_enable(on: bool):
    load().kblas_timing_enable(1 if on else 0)


def timing_read() -> tuple[float, int]:
    ms, n = c_double(0.0), c_int(0)
    check(load().kblas_timing_read(ctypes.byref(ms), ctypes.byref(n)), "kblas_timing_read")
    return ms.value, n.value
