"""Counter-based operand generator shared by the oracle and the tests
(TEST INFRASTRUCTURE only).

Large-N parity (BASELINE configs[1]-[4]: 8.6-160 GB operands) needs the
CPU oracle to see exactly the operand the GPU saw without a host copy.  So
the operand is a pure function of (seed, global row, global column), as
SURVEY §8c / BASELINE.md §3.3 ask ("regenerate the panel from (seed, block
col)"): oracle/streamed.c regenerates every stored element inside its
streamed loops, and `fill_*` below writes the same values into device
tensors with torch integer ops.  The definition (streamed.c header):

    u(k) = (splitmix64((seed << 36) + k) >> 11) * 2^-52 - 1      in [-1, 1)
    k = (j + co) * gen_ld + (i + ro)          real: a = u(k)
                                              complex: a = u(2k) + i u(2k+1)
    float / complex64 operands: the double value rounded to float.

Every step is exact in IEEE double (a 53-bit integer scaled by a power of
two, minus one), so numpy, torch (CPU or CUDA) and C agree bit for bit;
tests/test_oracle.py pins that.
"""

from __future__ import annotations

import numpy as np

C1 = 0x9E3779B97F4A7C15
C2 = 0xBF58476D1CE4E5B9
C3 = 0x94D049BB133111EB
M64 = (1 << 64) - 1


def _signed(c: int) -> int:
    return c - (1 << 64) if c >= 1 << 63 else c


# ----------------------------------------------------------------- numpy
def mix64_np(k: np.ndarray) -> np.ndarray:
    z = k.astype(np.uint64) + np.uint64(C1)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(C2)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(C3)
    return z ^ (z >> np.uint64(31))


def u_np(seed: int, k: np.ndarray) -> np.ndarray:
    h = mix64_np((np.uint64(seed) << np.uint64(36)) + k.astype(np.uint64))
    return (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -52 - 1.0


def values_np(tag: str, seed: int, keys: np.ndarray) -> np.ndarray:
    if tag in "cz":
        v = u_np(seed, 2 * keys) + 1j * u_np(seed, 2 * keys + 1)
        return v.astype(np.complex64 if tag == "c" else np.complex128)
    v = u_np(seed, keys)
    return v.astype(np.float32 if tag == "s" else np.float64)


def matrix_np(tag: str, m: int, n: int, seed: int, gen_ld: int, ro: int = 0, co: int = 0) -> np.ndarray:
    """The generated m x n operand at (ro, co) (small sizes; tests)."""
    i = np.arange(m, dtype=np.int64)[:, None] + ro
    j = np.arange(n, dtype=np.int64)[None, :] + co
    return values_np(tag, seed, j * gen_ld + i)


def vector_np(tag: str, n: int, seed: int) -> np.ndarray:
    return values_np(tag, seed, np.arange(n, dtype=np.int64))


# ----------------------------------------------------------------- torch
def _lsr(z, s: int):
    """Logical right shift of int64 two's-complement words."""
    return (z >> s) & ((1 << (64 - s)) - 1)


def _u_torch(seed: int, k):
    import torch

    z = k + ((seed << 36) + _signed(C1))
    z = (z ^ _lsr(z, 30)) * _signed(C2)
    z = (z ^ _lsr(z, 27)) * _signed(C3)
    z = z ^ _lsr(z, 31)
    return _lsr(z, 11).to(torch.float64) * 2.0 ** -52 - 1.0


def values_torch(tag: str, seed: int, keys):
    """keys: int64 tensor -> operand values of precision `tag` (same device)."""
    import torch

    if tag in "cz":
        v = torch.complex(_u_torch(seed, 2 * keys), _u_torch(seed, 2 * keys + 1))
        return v.to(torch.complex64) if tag == "c" else v
    v = _u_torch(seed, keys)
    return v.to(torch.float32) if tag == "s" else v


DT = {"s": "float32", "d": "float64", "c": "complex64", "z": "complex128"}


def fill_columns(cols, tag: str, seed: int, gen_ld: int, rows: int, col0: int = 0, ro: int = 0, co: int = 0,
                 tri: str | None = None, poison=float("nan"), block: int = 256):
    """Write logical columns col0 .. col0+ncols-1 of the generated operand
    into `cols`, a (ncols, ld) row-major tensor whose row b is one
    column-major column (rows [0, rows) are written, padding untouched).

    Logical element (i, c) has key (c + co) * gen_ld + (i + ro).  tri 'l'
    ('u') keeps only the stored triangle i >= c (i <= c) and sets the other
    triangle to `poison` (NaN by default), so a kernel that reads it cannot
    pass."""
    import torch

    dev = cols.device
    ncols = cols.shape[0]
    i = torch.arange(rows, dtype=torch.int64, device=dev)[None, :]
    for b0 in range(0, ncols, block):
        b1 = min(ncols, b0 + block)
        c = torch.arange(b0, b1, dtype=torch.int64, device=dev)[:, None] + col0
        v = values_torch(tag, seed, (c + co) * gen_ld + (i + ro))
        if tri is not None:
            bad = (i < c) if tri == "l" else (i > c)
            v = torch.where(bad, torch.full((), poison, dtype=v.dtype, device=dev), v)
        cols[b0:b1, :rows] = v
        del v


def vector_torch(tag: str, n: int, seed: int, device):
    import torch

    return values_torch(tag, seed, torch.arange(n, dtype=torch.int64, device=device))
