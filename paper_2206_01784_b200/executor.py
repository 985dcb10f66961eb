"""Executor and memory-operation ledger.

Mirrors onesweep.executor (executor.py:36-219).  On the GPU the thread pool is
replaced by the CUDA grid (tile tickets are an atomicAdd in the binning
kernel), so `Executor` keeps only what callers observe: the `workers`
attribute (accepted and ignored), the optional `stream`, and the ledger.

The ledger is filled analytically -- n element reads for the histogram,
n reads + n writes per binning pass (binning.py:268-272) -- plus the
schedule-dependent columns the kernels count on the device:
fast_path_tiles (short-circuit tiles) and counter_ops (2*radix status writes
per tile plus look-back reads, binning.py:195-198).  Device counters are
materialised lazily, so recording never forces a host synchronisation.
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass, field, replace

_LEDGER_KINDS = (
    "element_reads",
    "element_writes",
    "counter_ops",
    "copy_ops",
    "fast_path_tiles",
)


@dataclass
class LedgerCounts:
    """Counters for one phase (executor.py:36-50)."""

    element_reads: int = 0
    element_writes: int = 0
    counter_ops: int = 0
    copy_ops: int = 0
    fast_path_tiles: int = 0


@dataclass(frozen=True)
class MemOpLedger:
    """Immutable snapshot of per-phase counts (executor.py:52-87)."""

    phases: dict[str, LedgerCounts] = field(default_factory=dict)

    def phase(self, name: str) -> LedgerCounts:
        return self.phases.get(name, LedgerCounts())

    def _total(self, kind: str) -> int:
        return sum(getattr(c, kind) for c in self.phases.values())

    @property
    def element_reads(self) -> int:
        return self._total("element_reads")

    @property
    def element_writes(self) -> int:
        return self._total("element_writes")

    @property
    def counter_ops(self) -> int:
        return self._total("counter_ops")

    @property
    def copy_ops(self) -> int:
        return self._total("copy_ops")

    @property
    def fast_path_tiles(self) -> int:
        return self._total("fast_path_tiles")

    @property
    def element_ops(self) -> int:
        return self.element_reads + self.element_writes


class Jitter:
    """Accepted for signature compatibility (executor.py:108-121).

    Block scheduling on the GPU is the hardware's; schedule exploration is done
    by the device tests (reverse tile-claim pressure, many small tiles)."""

    def __init__(self, seed: int = 0, max_pause_us: float = 50.0):
        self.seed = seed
        self.max_pause_us = max_pause_us

    def pause(self) -> None:  # pragma: no cover - nothing to pause on the host
        return None


class TileTicket:
    """Shared monotone counter issuing each tile index in [0, tiles) exactly
    once (executor.py:88-105).  The device kernels take their tile ids from an
    atomicAdd on a ticket word (csrc/binning.cu); this host twin keeps the
    reference's API for callers that schedule their own work."""

    def __init__(self, tiles: int):
        self._tiles = tiles
        self._next = 0
        self._lock = threading.Lock()

    def next_tile(self) -> int | None:
        """Next tile index, or None once all tiles have been issued."""
        with self._lock:
            if self._next >= self._tiles:
                return None
            tile = self._next
            self._next += 1
            return tile


class Executor:
    """Ledger owner for device sorts (executor.py:124-156)."""

    def __init__(self, workers: int | None = None, jitter: Jitter | None = None, stream=None):
        if workers is None:
            workers = os.cpu_count() or 1
        if workers < 1:
            raise ValueError(f"workers must be >= 1, got {workers}")
        self.workers = workers
        self.jitter = jitter
        self.stream = stream
        self._ledger: dict[str, LedgerCounts] = {}
        # element reads + writes the device actually performed (equal to the
        # ledger's element_ops except when cfg.digit_bits > 8 runs as 8-bit places)
        self.device_element_ops = 0
        self._pending: list[tuple[str, object, int]] = []  # (phase, device stats, radix)
        self._lock = threading.Lock()

    def ledger_record(self, phase: str, kind: str, count: int) -> None:
        if kind not in _LEDGER_KINDS:
            raise ValueError(f"unknown ledger kind {kind!r}")
        with self._lock:
            counts = self._ledger.setdefault(phase, LedgerCounts())
            setattr(counts, kind, getattr(counts, kind) + int(count))

    def record_device_stats(self, phase: str, stats, radix: int) -> None:
        """Queue an os_device_stats tensor [fast_tiles, lookback_reads, tiles]."""
        with self._lock:
            self._pending.append((phase, stats, radix))

    def _drain(self) -> None:
        pending, self._pending = self._pending, []
        for phase, stats, radix in pending:
            fast, reads, tiles = (int(x) for x in stats.view(__import__("torch").int64).tolist()[:3])
            counts = self._ledger.setdefault(phase, LedgerCounts())
            counts.fast_path_tiles += fast
            counts.counter_ops += 2 * radix * tiles + reads

    def ledger_snapshot(self) -> MemOpLedger:
        with self._lock:
            self._drain()
            return MemOpLedger(phases={k: replace(v) for k, v in self._ledger.items()})

    def ledger_reset(self) -> None:
        with self._lock:
            self._ledger.clear()
            self._pending.clear()
            self.device_element_ops = 0


def ledger_as_row(ledger: MemOpLedger) -> dict[str, int]:
    """Flatten ledger totals into the bench CSV columns (executor.py:215-219)."""
    row = {kind: getattr(ledger, kind) for kind in _LEDGER_KINDS}
    row["element_ops"] = ledger.element_ops
    return row


__all__ = ["Executor", "Jitter", "LedgerCounts", "MemOpLedger", "TileTicket", "ledger_as_row"]
