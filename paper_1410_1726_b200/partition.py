"""KernelConfig and the balanced split used for cooperating work shares.

`KernelConfig` keeps the reference's validation (partition.py:25-36) so
existing call sites construct it unchanged.  On B200 the triple is a
tuning hint only: the kernels pick their own tile shape for sm_100a
(csrc/kblas_impl.cuh, `Cfg`), and the cooperating-TB split-K of the paper
(Y-bar) is replaced by stream-K over equal work items.  `block_size` still
matters for the mgpu SYMV/HEMV distribution check (multidevice.py:205-208).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class KernelConfig:
    """(nb, Q-bar, Y-bar) tuning triple (partition.py:13-45)."""

    block_size: int
    thread_cols: int
    coop_tbs: int = 1

    def __post_init__(self):
        if self.block_size <= 0 or self.block_size % 2 != 0:
            raise ValueError(f"block_size must be positive and even, got {self.block_size}")
        if self.thread_cols <= 0:
            raise ValueError(f"thread_cols must be positive, got {self.thread_cols}")
        if self.coop_tbs < 1:
            raise ValueError(f"coop_tbs must be >= 1, got {self.coop_tbs}")
        if self.block_size % (2 * self.thread_cols) != 0:
            raise ValueError(
                f"block_size/(2*thread_cols) must be a positive integer "
                f"(got {self.block_size}/{2 * self.thread_cols})"
            )

    @property
    def buffer_len(self) -> int:
        return self.block_size // (2 * self.thread_cols)

    @property
    def threads_per_tb(self) -> int:
        return self.block_size * self.thread_cols


DEFAULT_CONFIG = KernelConfig(64, 4, 1)


def tb_share(total: int, coop_tbs: int, slot: int) -> tuple[int, int]:
    """(workload, start) of slot `slot` among `coop_tbs` (partition.py:101-114)."""
    if total < 0:
        raise ValueError(f"total workload must be >= 0, got {total}")
    if not 0 <= slot < coop_tbs:
        raise ValueError(f"slot {slot} out of range for {coop_tbs} cooperating TBs")
    base, rem = divmod(total, coop_tbs)
    w = base + (1 if slot < rem else 0)
    s = slot * base + min(slot, rem)
    return w, s


def sk_start(c: int, total: int, p: int) -> int:
    """First item of CTA c under the stream-K split (csrc/kblas_device.cuh)."""
    return c * total // p


def sk_owner(i: int, total: int, p: int) -> int:
    """CTA owning item i under the stream-K split."""
    return ((i + 1) * p - 1) // total
