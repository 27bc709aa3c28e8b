"""Multiply-add accounting shim (behaviour of `pkg/src/hbs/flops.py:19-55`).

The device path does not count work per node; instead the host charges, per
level, exactly the nominal madds the reference's per-node calls would have
charged (same shape formulas), so machine-independent cost tests keep working
against the drop-in.
"""

from contextlib import contextmanager
from contextvars import ContextVar
from dataclasses import dataclass


@dataclass
class MaddCounter:
    madds: int = 0


_COUNTER: ContextVar = ContextVar("hbs_b200_madds", default=None)


@contextmanager
def count_madds():
    """Activate a counter for the dynamic extent of the block (flops.py:22-30)."""
    counter = MaddCounter()
    token = _COUNTER.set(counter)
    try:
        yield counter
    finally:
        _COUNTER.reset(token)


def counting() -> bool:
    return _COUNTER.get() is not None


def add_madds(n) -> None:
    counter = _COUNTER.get()
    if counter is not None:
        counter.madds += int(n)


def matmul_madds(m, k, n):
    """(m x k) @ (k x n) (flops.py:39-41)."""
    return m * k * n


def qr_madds(m, n, full=False):
    """Householder QR of m x n (m >= n) plus explicit Q (flops.py:44-49)."""
    return m * n * n - n ** 3 // 3 + (m * m * n if full else m * n * n)


def svd_madds(m, n):
    """Coarse thin-SVD count (flops.py:52-55)."""
    k = min(m, n)
    return 2 * m * n * k + 4 * k ** 3


def node_compress_madds(rows: int, s: int, r: int) -> int:
    """Madds the reference charges for one non-root node's bases and
    discrepancy: `compress.py:169-174` (nullspace + product + col, both sides)
    and `compress.py:192-194` (two lstsq_right solves + projector algebra)."""
    bases = 2 * (qr_madds(s, rows, full=True) + matmul_madds(rows, s, r) + qr_madds(rows, r))
    solve = 2 * (svd_madds(rows, s) + matmul_madds(rows, s, rows) + matmul_madds(rows, rows, rows))
    return bases + solve + 6 * matmul_madds(r, rows, rows)


def lift_madds(rows: int, s: int, r: int) -> int:
    """Madds charged per child by `lift_to_parent` (compress.py:213)."""
    return 4 * matmul_madds(r, rows, s) + 2 * matmul_madds(rows, rows, s)


def root_madds(rows: int, s: int) -> int:
    """`compute_root` = one lstsq_right (linalg.py:81,89)."""
    return svd_madds(rows, s) + matmul_madds(rows, s, rows) + matmul_madds(rows, rows, rows)
