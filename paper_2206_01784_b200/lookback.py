"""Chained-scan status words (lookback.py:1-189), device edition.

The binning kernel publishes and reads the reference's exact word format --
bits 31-30 status {N=0, L=1, G=2}, bits 29-0 value -- in a tile-major
u32[tiles][radix] array (lookback.py:63-79).  The protocol itself runs inside
csrc/binning.cu; this module keeps the word helpers, a view of a finished
pass's words, and a host model of the protocol for single-tile callers.
"""

from __future__ import annotations

import time

import numpy as np

STATUS_NOT_READY = 0  # N
STATUS_LOCAL = 1  # L
STATUS_GLOBAL = 2  # G

STATUS_SHIFT = 30
VALUE_MASK = (1 << STATUS_SHIFT) - 1
MAX_COUNTER_VALUE = VALUE_MASK


class LookbackAborted(RuntimeError):
    """A host-side look-back gave up waiting on a predecessor (lookback.py:45-46)."""


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


_SPIN_YIELDS = 64  # polls that only yield before a waiter starts sleeping


class CounterMatrix:
    """One strip's status words, tile-major u32[tiles][radix] (lookback.py:63-79).

    Two uses:
    * ``CounterMatrix(words)`` wraps the final words a device pass left behind
      (``partition_pass(..., return_status=True)``) for inspection;
    * ``CounterMatrix(tiles, radix[, abort_event])`` is a zeroed host model of
      the protocol for callers that drive single tiles (``process_tile``) or
      exercise the protocol itself: N -> L -> G publishes with the same
      transition checks, and the look-back walk that sums L values down to
      the first G (lookback.py:81-176).  The sort never uses the host model:
      the device kernel runs the protocol on its own status array
      (csrc/binning.cu, step 4b)."""

    def __init__(self, tiles, radix: int | None = None, abort_event=None):
        if radix is None:
            self.words = np.asarray(tiles, dtype=np.uint32)
        else:
            self.words = np.zeros((int(tiles), int(radix)), dtype=np.uint32)
        self.tiles, self.radix = self.words.shape
        self.abort_event = abort_event

    # -- single counters ----------------------------------------------------
    def load(self, digit: int, tile: int) -> int:
        return int(self.words[tile, digit])

    def _status(self, digit: int, tile: int) -> int:
        return self.load(digit, tile) >> STATUS_SHIFT

    def publish_local(self, digit: int, tile: int, local_count: int) -> None:
        assert self._status(digit, tile) == STATUS_NOT_READY, f"L published twice: tile {tile} digit {digit}"
        self.words[tile, digit] = pack_counter(STATUS_LOCAL, int(local_count))

    def publish_inclusive(self, digit: int, tile: int, inclusive: int) -> None:
        assert self._status(digit, tile) == STATUS_LOCAL, f"G before L: tile {tile} digit {digit}"
        self.words[tile, digit] = pack_counter(STATUS_GLOBAL, int(inclusive))

    def lookback_exclusive(self, digit: int, tile: int) -> int:
        exclusive, _ = self._walk(tile, np.array([digit]))
        return int(exclusive[0])

    # -- whole rows ---------------------------------------------------------
    def publish_local_row(self, tile: int, local_counts) -> None:
        row = np.asarray(local_counts, dtype=np.int64)
        if row.size and (row.min() < 0 or row.max() > MAX_COUNTER_VALUE):
            raise ValueError("local count does not fit in 30 bits")
        assert not self.words[tile].any(), f"L row published twice: tile {tile}"
        self.words[tile] = row.astype(np.uint32) | np.uint32(STATUS_LOCAL << STATUS_SHIFT)

    def publish_inclusive_row(self, tile: int, inclusive) -> None:
        row = np.asarray(inclusive, dtype=np.int64)
        if row.size and (row.min() < 0 or row.max() > MAX_COUNTER_VALUE):
            raise ValueError("inclusive prefix does not fit in 30 bits")
        self.words[tile] = row.astype(np.uint32) | np.uint32(STATUS_GLOBAL << STATUS_SHIFT)

    def lookback_exclusive_row(self, tile: int) -> tuple[np.ndarray, int]:
        """(exclusive prefix per digit as int64, status words read)."""
        return self._walk(tile, np.arange(self.radix))

    def _walk(self, tile: int, digits: np.ndarray) -> tuple[np.ndarray, int]:
        exclusive = np.zeros(digits.size, dtype=np.int64)
        open_ = np.arange(digits.size)  # positions still walking
        reads = polls = 0
        j = tile - 1
        while j >= 0 and open_.size:
            words = self.words[j, digits[open_]]
            reads += open_.size
            status = words >> np.uint32(STATUS_SHIFT)
            if (status == STATUS_NOT_READY).any():  # a predecessor is in flight
                polls += 1
                self._wait(polls)
                continue
            exclusive[open_] += (words & np.uint32(VALUE_MASK)).astype(np.int64)
            open_ = open_[status == STATUS_LOCAL]  # a G word ends that digit's walk
            j -= 1
        return exclusive, reads

    def _wait(self, polls: int) -> None:
        if self.abort_event is not None and self.abort_event.is_set():
            raise LookbackAborted("look-back aborted while a predecessor was unpublished")
        time.sleep(0 if polls < _SPIN_YIELDS else 1e-4)

    def final_inclusive(self, digit: int | None = None):
        if digit is None:
            return (self.words[self.tiles - 1] & np.uint32(VALUE_MASK)).astype(np.int64)
        return self.load(digit, self.tiles - 1) & VALUE_MASK
