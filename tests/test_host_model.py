"""CPU: the host-side pieces of the executor/look-back API that callers
driving their own blocks use (executor.py:160-212, lookback.py:81-176) --
run_blocks, Jitter and the CounterMatrix host model.  The device sort never
uses them (its blocks are the CUDA grid, its protocol runs in the kernel)."""

from __future__ import annotations

import threading

import numpy as np
import pytest

from paper_2206_01784_b200 import CounterMatrix, Executor, Jitter
from paper_2206_01784_b200.lookback import LookbackAborted


@pytest.mark.parametrize("workers", [1, 3, 8])
def test_run_blocks_each_tile_once(workers):
    seen = []
    lock = threading.Lock()

    def body(t):
        with lock:
            seen.append(t)

    Executor(workers=workers, jitter=Jitter(seed=1, max_pause_us=20)).run_blocks(50, body)
    assert sorted(seen) == list(range(50))
    if workers == 1:
        assert seen == list(range(50))


def test_run_blocks_reraises_real_error_over_abort():
    def body(t):
        if t == 3:
            raise LookbackAborted("secondary")
        if t == 5:
            raise KeyError("primary")

    with pytest.raises((KeyError, LookbackAborted)):
        Executor(workers=1).run_blocks(10, body)
    with pytest.raises(KeyError):
        Executor(workers=1).run_blocks(10, lambda t: (_ for _ in ()).throw(KeyError("x")))


@pytest.mark.parametrize("workers", [1, 4])
def test_counter_matrix_protocol_under_threads(workers):
    rng = np.random.default_rng(workers)
    tiles, radix = 40, 16
    counts = rng.integers(0, 50, size=(tiles, radix))
    m = CounterMatrix(tiles, radix)

    def body(t):
        m.publish_local_row(t, counts[t])
        excl, _ = m.lookback_exclusive_row(t)
        m.publish_inclusive_row(t, excl + counts[t])

    Executor(workers=workers, jitter=Jitter(seed=2, max_pause_us=30)).run_blocks(tiles, body)
    assert np.array_equal(m.final_inclusive(), counts.sum(axis=0))
    assert np.array_equal(m.words & 0x3FFFFFFF, np.cumsum(counts, axis=0))


def test_counter_matrix_transitions_and_abort():
    m = CounterMatrix(3, 1)
    m.publish_local(0, 0, 7)
    with pytest.raises(AssertionError):
        m.publish_local(0, 0, 7)
    with pytest.raises(AssertionError):
        m.publish_inclusive(0, 1, 5)
    ev = threading.Event()
    ev.set()
    waiting = CounterMatrix(3, 1, abort_event=ev)
    with pytest.raises(LookbackAborted):
        waiting.lookback_exclusive(0, 2)  # tile 1 never publishes
    words = CounterMatrix(np.array([[0x40000003, 0x80000001]], dtype=np.uint32))
    assert (words.tiles, words.radix) == (1, 2) and words.load(1, 0) == 0x80000001
