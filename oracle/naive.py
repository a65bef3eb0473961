"""numpy restatement of the reference oracle (blockmv/reference.py:15-70)
and of the reference's input generators.  Test infrastructure only."""

from __future__ import annotations

import numpy as np

DTYPES = {"s": np.float32, "d": np.float64, "c": np.complex64, "z": np.complex128}
EPS = {"s": float(np.finfo(np.float32).eps), "c": float(np.finfo(np.float32).eps),
       "d": float(np.finfo(np.float64).eps), "z": float(np.finfo(np.float64).eps)}


def wide(arr):
    """reference.py:15-16: f64 / c128 working precision."""
    arr = np.asarray(arr)
    return arr.astype(np.complex128 if np.iscomplexobj(arr) else np.float64)


def dense_from_triangle(a2d, uplo: str, hermitian: bool):
    """reference.py:19-36: full matrix from one stored triangle; Hermitian
    mirrors the conjugate and forces a real diagonal."""
    a = wide(a2d)
    if uplo == "l":
        tri, mirror = np.tril(a), np.tril(a, -1)
    else:
        tri, mirror = np.triu(a), np.triu(a, 1)
    full = tri + (mirror.conj().T if hermitian else mirror.T)
    if hermitian:
        idx = np.arange(full.shape[0])
        full[idx, idx] = full[idx, idx].real
    return full


def naive_gemv(trans: str, alpha, a2d, x, beta, y, out_dtype=None):
    """reference.py:39-50."""
    mat = wide(a2d)
    trans = trans.lower()
    if trans == "t":
        mat = mat.T
    elif trans == "c":
        mat = mat.conj().T
    elif trans != "n":
        raise ValueError(f"trans must be 'n', 't' or 'c', got {trans!r}")
    xw, yw = wide(x), wide(y)
    out = alpha * (mat @ xw) + (beta * yw if beta != 0 else 0.0)
    return out.astype(out_dtype or np.asarray(a2d).dtype)


def naive_symv_hemv(alpha, a2d, uplo: str, x, beta, y, hermitian: bool | None = None, out_dtype=None):
    """reference.py:53-59."""
    a2d = np.asarray(a2d)
    if hermitian is None:
        hermitian = np.iscomplexobj(a2d)
    full = dense_from_triangle(a2d, uplo, hermitian)
    xw, yw = wide(x), wide(y)
    out = alpha * (full @ xw) + (beta * yw if beta != 0 else 0.0)
    return out.astype(out_dtype or a2d.dtype)


def tolerance_bound(a_abs, x, tag: str, factor: float = 50.0) -> float:
    """reference.py:62-66: factor * eps * ||A||_inf * ||x||_inf."""
    a_abs = np.asarray(a_abs)
    norm_a = float(np.max(np.sum(np.abs(a_abs), axis=1))) if a_abs.size else 0.0
    norm_x = float(np.max(np.abs(np.asarray(x)))) if len(x) else 0.0
    return factor * EPS[tag] * norm_a * norm_x


def max_abs_error(got, want) -> float:
    """reference.py:69-70."""
    return float(np.max(np.abs(np.asarray(got) - np.asarray(want))))


def run_bound(tag: str, alpha, a_abs_dense, x, beta, y) -> float:
    """The blockmv CLI verify bound (cli.py:171-175):
    50 eps (|alpha| ||A|| ||x|| + |beta| ||y||)."""
    return tolerance_bound(abs(alpha) * np.abs(a_abs_dense), x, tag) + tolerance_bound(
        abs(beta) * np.eye(len(y)), y, tag)


# ------------------------------------------------------------ generators
def fill(rng, shape, tag: str):
    """cli.py:52-57: U(-1, 1), complex with independent re/im."""
    if tag in "cz":
        re = rng.uniform(-1, 1, size=shape)
        im = rng.uniform(-1, 1, size=shape)
        return (re + 1j * im).astype(DTYPES[tag])
    return rng.uniform(-1, 1, size=shape).astype(DTYPES[tag])


def signed_uniform(rng, shape, tag: str):
    """test_acceptance.py:37-45: magnitudes in [0.5, 1) with random signs."""
    mag = rng.uniform(0.5, 1.0, shape)
    sign = rng.choice([-1.0, 1.0], shape)
    if tag in "cz":
        mag_i = rng.uniform(0.5, 1.0, shape)
        sign_i = rng.choice([-1.0, 1.0], shape)
        return (mag * sign + 1j * mag_i * sign_i).astype(DTYPES[tag])
    return (mag * sign).astype(DTYPES[tag])


def random_matrix(rng, m: int, n: int, tag: str, pad_to: int = 32):
    """test_kernels.py:21-29: flat column-major buffer, ld padded to 32.
    Returns (flat, ld); the (m, n) window is flat[:ld*n].reshape(n, ld).T[:m]."""
    ld = -(-m // pad_to) * pad_to
    flat = np.zeros(ld * n, dtype=DTYPES[tag])
    win = flat.reshape(n, ld).T[:m]
    if tag in "cz":
        win[:, :] = rng.uniform(-1, 1, (m, n)) + 1j * rng.uniform(-1, 1, (m, n))
    else:
        win[:, :] = rng.uniform(-1, 1, (m, n))
    return flat, ld


def window(flat, ld: int, m: int, n: int, row_off: int = 0, col_off: int = 0):
    """(m, n) column-major window of a flat buffer (core.py:100-101,120-132)."""
    start = col_off * ld + row_off
    item = flat.itemsize
    return np.lib.stride_tricks.as_strided(flat[start:], shape=(m, n), strides=(item, ld * item))


def random_vec(rng, n: int, tag: str):
    """test_kernels.py:32-36."""
    if tag in "cz":
        return (rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)).astype(DTYPES[tag])
    return rng.uniform(-1, 1, n).astype(DTYPES[tag])
