"""Chained-scan status words (lookback.py:1-189), device edition.

The binning kernel publishes and reads the reference's exact word format --
bits 31-30 status {N=0, L=1, G=2}, bits 29-0 value -- in a tile-major
u32[tiles][radix] array (lookback.py:63-79).  The protocol itself runs inside
csrc/binning.cu; this module keeps the word helpers and a read-only view of a
finished pass's words for inspection and parity tests.
"""

from __future__ import annotations

import numpy as np

STATUS_NOT_READY = 0  # N
STATUS_LOCAL = 1  # L
STATUS_GLOBAL = 2  # G

STATUS_SHIFT = 30
VALUE_MASK = (1 << STATUS_SHIFT) - 1
MAX_COUNTER_VALUE = VALUE_MASK


class LookbackAborted(RuntimeError):
    """Kept for API compatibility (lookback.py:45-46); device passes cannot abort."""


def pack_counter(status: int, value: int) -> int:
    """Pack (status, value) into one 32-bit word (lookback.py:49-55)."""
    if status not in (STATUS_NOT_READY, STATUS_LOCAL, STATUS_GLOBAL):
        raise ValueError(f"invalid status {status}")
    if not 0 <= value <= MAX_COUNTER_VALUE:
        raise ValueError(f"counter value {value} does not fit in 30 bits")
    return (status << STATUS_SHIFT) | value


def unpack_counter(word: int) -> tuple[int, int]:
    """Exact inverse of pack_counter (lookback.py:58-60)."""
    return (word >> STATUS_SHIFT) & 0x3, word & VALUE_MASK


class CounterMatrix:
    """Read-only view of one strip's final status words.

    `words` is a (tiles, radix) uint32 numpy array copied from the device
    after the pass; the query methods mirror lookback.py:81-83,171-176."""

    def __init__(self, words: np.ndarray):
        self.words = np.asarray(words, dtype=np.uint32)
        self.tiles, self.radix = self.words.shape

    def load(self, digit: int, tile: int) -> int:
        return int(self.words[tile, digit])

    def final_inclusive(self, digit: int | None = None):
        if digit is None:
            return (self.words[self.tiles - 1] & np.uint32(VALUE_MASK)).astype(np.int64)
        return self.load(digit, self.tiles - 1) & VALUE_MASK
