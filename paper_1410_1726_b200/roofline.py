"""Algorithmic flop / byte counts: the numerators of Gflop/s and GB/s.

Square forms restate blockmv/roofline.py:20-42; the rectangular and
submatrix forms follow SURVEY.md §8(d): only the true (sub)matrix, x once,
y read and written once.  Alignment padding and masked lead rows are never
credited.
"""

from __future__ import annotations

from .core import Precision

FAMILIES = ("gemv", "symv")


def flop_count(prec: Precision, family: str, n: int) -> int:
    """(n^2 + 2n) multiplies and n^2 adds (roofline.py:20-32)."""
    if family not in FAMILIES:
        raise ValueError(f"unknown kernel family {family!r}")
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    return prec.flops_per_mul * (n * n + 2 * n) + prec.flops_per_add * n * n


def byte_count(prec: Precision, family: str, n: int) -> int:
    """gemv (n^2 + 3n) b, symv (n(n+1)/2 + 3n) b (roofline.py:35-42)."""
    if family == "gemv":
        return (n * n + 3 * n) * prec.element_bytes
    if family == "symv":
        return (n * (n + 1) // 2 + 3 * n) * prec.element_bytes
    raise ValueError(f"unknown kernel family {family!r}")


def gemv_bytes(prec: Precision, m: int, n: int, trans: str = "n") -> int:
    """b (m n + len(x) + 2 len(y))."""
    x_len, y_len = (n, m) if trans.lower() == "n" else (m, n)
    return (m * n + x_len + 2 * y_len) * prec.element_bytes


def symv_bytes(prec: Precision, d: int) -> int:
    return (d * (d + 1) // 2 + 3 * d) * prec.element_bytes


def gemv_flops(prec: Precision, m: int, n: int, trans: str = "n") -> int:
    """mul (mn + 2 len(y)) + add mn: product, alpha, beta (kernels.py:204-206 + run_scal)."""
    y_len = m if trans.lower() == "n" else n
    return prec.flops_per_mul * (m * n + 2 * y_len) + prec.flops_per_add * m * n


def symv_flops(prec: Precision, d: int) -> int:
    return prec.flops_per_mul * (d * d + 2 * d) + prec.flops_per_add * d * d


ROOFLINE_CSV_HEADER = ["precision", "family", "n", "flops", "bytes", "intensity", "peak_gflops", "note"]


def write_intensity_csv(fh, copy_peak_gbs: float, source: str, sample_n: int = 1_000_000) -> None:
    """The intensity / bandwidth-bound table of blockmv/roofline.py:92-136
    for the B200: all 4 precisions x 2 families, intensity exact at
    sample_n, peak = intensity x the measured copy bandwidth (the roofline
    every kernel here is bound by)."""
    import csv

    from .core import precision

    w = csv.writer(fh)
    w.writerow(ROOFLINE_CSV_HEADER)
    for tag in "sdcz":
        prec = precision(tag)
        for family in FAMILIES:
            f, b = flop_count(prec, family, sample_n), byte_count(prec, family, sample_n)
            w.writerow([tag, family, sample_n, f, b, f"{f / b:.6f}", f"{f / b * copy_peak_gbs:.2f}",
                        f"copy peak {copy_peak_gbs:.1f} GB/s ({source})"])
