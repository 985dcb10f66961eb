"""Executor and memory-operation ledger.

Mirrors onesweep.executor (executor.py:36-219).  On the GPU the thread pool is
replaced by the CUDA grid (tile tickets are an atomicAdd in the binning
kernel); `Executor` keeps what callers observe -- `workers`, the optional
`stream`, the ledger -- and `run_blocks` for host-driven blocks only.

The ledger is filled analytically -- n element reads for the histogram,
n reads + n writes per binning pass (binning.py:268-272) -- plus the
schedule-dependent columns the kernels count on the device:
fast_path_tiles (short-circuit tiles) and counter_ops (2*radix status writes
per tile plus look-back reads, binning.py:195-198).  Device counters are
materialised lazily, so recording never forces a host synchronisation.
"""

from __future__ import annotations

import os
import random
import threading
import time
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
    """Seeded random pauses around host-driven blocks (executor.py:108-121).

    Device passes explore schedules with the debug library's in-kernel
    __nanosleep jitter instead (tests/test_gpu_race.py)."""

    def __init__(self, seed: int = 0, max_pause_us: float = 50.0):
        self.seed = seed
        self.max_pause_us = max_pause_us
        self._tls = threading.local()

    def pause(self) -> None:
        """Sleep a seeded pseudo-random 0..max_pause_us (per-thread stream);
        used by Executor.run_blocks around host-driven blocks."""
        gen = getattr(self._tls, "gen", None)
        if gen is None:
            gen = self._tls.gen = random.Random(hash((self.seed, threading.get_ident())))
        time.sleep(gen.random() * self.max_pause_us * 1e-6)


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
        self._device_ops = 0
        self._pending_routes: list[tuple[int, object]] = []  # (n, route words) of os_sort calls
        self._pending: list[tuple[str, object, int]] = []  # (phase, device stats, radix)
        self._lock = threading.Lock()

    def run_blocks(self, tiles: int, body) -> None:
        """Host dispatch of body(tile) for tile in [0, tiles) on `workers`
        threads (executor.py:160-212): ids come from one TileTicket in
        increasing order, a thread finishes a block before drawing the next,
        all threads are joined before returning, and the first failure is
        re-raised (a real error in preference to a LookbackAborted it caused).
        The device sort never calls this -- its blocks are the CUDA grid; it
        serves callers that drive host-side blocks (process_tile)."""
        if tiles <= 0:
            return
        ticket = TileTicket(tiles)
        halt = threading.Event()
        errors: list[BaseException] = []

        def drain() -> None:
            while not halt.is_set() and (tile := ticket.next_tile()) is not None:
                try:
                    if self.jitter is not None:
                        self.jitter.pause()
                    body(tile)
                    if self.jitter is not None:
                        self.jitter.pause()
                except BaseException as exc:  # noqa: BLE001 - re-raised below
                    errors.append(exc)
                    halt.set()

        if self.workers == 1:
            drain()
        else:
            pool = [threading.Thread(target=drain, name=f"onesweep-block-{i}")
                    for i in range(self.workers)]
            for t in pool:
                t.start()
            for t in pool:
                t.join()
        if errors:
            from .lookback import LookbackAborted

            raise next((e for e in errors if not isinstance(e, LookbackAborted)), errors[0])

    def ledger_record(self, phase: str, kind: str, count: int) -> None:
        if kind not in _LEDGER_KINDS:
            raise ValueError(f"unknown ledger kind {kind!r}")
        with self._lock:
            counts = self._ledger.setdefault(phase, LedgerCounts())
            setattr(counts, kind, getattr(counts, kind) + int(count))

    @property
    def device_element_ops(self) -> int:
        """Element reads + writes the device performed: the ledger's
        element_ops, except for places the device skipped (one bin held every
        key) and cfg.digit_bits > 8 plans run as 8-bit places."""
        with self._lock:
            pending, self._pending_routes = self._pending_routes, []
        for n, words in pending:
            from .binning import skipped_from_route_words

            skipped = skipped_from_route_words(words)
            self._device_ops += (1 + 2 * (len(skipped) - sum(skipped))) * n
        return self._device_ops

    @device_element_ops.setter
    def device_element_ops(self, value: int) -> None:
        with self._lock:
            self._pending_routes = []
        self._device_ops = int(value)

    def record_device_route(self, n: int, words) -> None:
        """Queue the route words of an os_sort of n keys (see device_element_ops)."""
        with self._lock:
            self._pending_routes.append((int(n), words))

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
            self._pending_routes.clear()
            self._device_ops = 0


def ledger_as_row(ledger: MemOpLedger) -> dict[str, int]:
    """Flatten ledger totals into the bench CSV columns (executor.py:215-219)."""
    row = {kind: getattr(ledger, kind) for kind in _LEDGER_KINDS}
    row["element_ops"] = ledger.element_ops
    return row


__all__ = ["Executor", "Jitter", "LedgerCounts", "MemOpLedger", "TileTicket", "ledger_as_row"]
