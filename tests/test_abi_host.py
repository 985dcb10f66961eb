"""CPU: the C-ABI library loads and exports every header symbol; host-side
logic (validation, error mapping, planning, ledger) behaves like the reference.
No kernel is launched here."""

from __future__ import annotations

import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "onesweep_b200.h")


def header_symbols() -> list[str]:
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(os_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2206_01784_b200 import _native

    lib = _native.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    # and the Python binding declares a signature for each of them
    assert set(syms) == set(_native.SIGNATURES)


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump -lelf {_lib_path()} 2>&1").read()
    assert "sm_100a" in out


def _lib_path():
    from paper_2206_01784_b200 import _native

    return _native.LIB_PATH


def test_host_only_entry_points():
    from paper_2206_01784_b200 import _native

    L = _native.load()
    assert b"sm_100a" in L.os_version()
    assert L.os_max_digit_bits() == 8
    assert L.os_tile_capacity(4, 0) >= 4096
    assert L.os_tile_capacity(8, 8) >= 2048
    assert L.os_tile_capacity(3, 0) == 0
    ws = L.os_sort_workspace_bytes(1 << 20, 0, 0, 8, 0, 32, 0, 0)
    assert ws >= 4 * (1 << 20)  # at least the ping-pong key buffer
    assert L.os_sort_workspace_bytes(100, 9, 0, 8, 0, 32, 0, 0) == 0  # bad key type
    assert L.os_sort_workspace_bytes(100, 0, 0, 9, 0, 32, 0, 0) == 0  # digit too wide
    assert L.os_sort_workspace_bytes(100, 0, 3, 8, 0, 32, 0, 0) == 0  # bad value width
    words = L.os_partition_status_words(10_000, 4, 64, 1000)
    assert words == (10 * 16) * 16  # 10 strips x 16 tiles x radix 16


def test_error_mapping():
    from paper_2206_01784_b200 import _native

    L = _native.load()
    rc = L.os_keygen(None, 0, 48, 1, 0, 0, None)
    with pytest.raises(ValueError, match="key_bits"):
        _native.check(rc)
    rc = L.os_encode(None, None, 0, 42, None)
    with pytest.raises(KeyError):
        _native.check(rc)


def test_radix_plan_validation_matches_reference():
    from paper_2206_01784_b200 import radix_plan

    cfg = radix_plan(32, 8, 4096)
    assert (cfg.passes, cfg.radix) == (4, 256)
    assert radix_plan(32, 7).passes == 5 and radix_plan(64, 8).passes == 8
    for bad in [dict(key_bits=32, digit_bits=0), dict(key_bits=32, digit_bits=17),
                dict(key_bits=32, digit_bits=8, tile_size=1 << 30),
                dict(key_bits=32, digit_bits=8, tile_size=0),
                dict(key_bits=32, digit_bits=8, strip_size=0),
                dict(key_bits=48, digit_bits=8),
                dict(key_bits=32, digit_bits=8, strip_size=(1 << 28) + 1)]:
        with pytest.raises(ValueError):
            radix_plan(**bad)
    with pytest.raises(ValueError):
        radix_plan(32, 8).digit_shift(4)


def test_key_type_lookup():
    from paper_2206_01784_b200 import key_spec, spec_for_dtype

    with pytest.raises(KeyError):
        key_spec("u16")
    with pytest.raises(KeyError):
        spec_for_dtype(np.dtype(np.float16))
    import torch

    assert spec_for_dtype(torch.uint32).name == "u32"
    assert spec_for_dtype(np.float64).name == "f64"


def test_sort_argument_errors_before_device():
    # binning.py:289-304 / test_binning.py:399-405 -- raised before any launch
    from paper_2206_01784_b200 import onesweep_sort, radix_plan

    with pytest.raises(KeyError):
        onesweep_sort(np.zeros(4, dtype=np.float16))
    with pytest.raises(ValueError):
        onesweep_sort(np.zeros(4, dtype=np.uint32), cfg=radix_plan(64, 8))
    with pytest.raises(ValueError):
        onesweep_sort(np.zeros(4, dtype=np.uint32), np.zeros(3, dtype=np.uint32))
    with pytest.raises(ValueError):
        onesweep_sort(np.zeros(4, dtype=np.uint32), begin_bit=8, end_bit=8)


def test_sort_trivial_sizes_return_copies():
    # binning.py:306-309 -- n <= 1 returns copies without touching the device
    from paper_2206_01784_b200 import onesweep_sort

    empty = onesweep_sort(np.empty(0, dtype=np.uint32))
    assert empty.size == 0 and empty.dtype == np.uint32
    src = np.array([42], dtype=np.uint32)
    one = onesweep_sort(src)
    assert one.tolist() == [42] and one is not src
    k, v = onesweep_sort(np.array([7], dtype=np.uint32), np.array([9], dtype=np.uint64))
    assert k.tolist() == [7] and v.tolist() == [9]


def test_counter_words():
    # test_lookback.py:30-33, 36-47
    from paper_2206_01784_b200.lookback import (STATUS_GLOBAL, STATUS_LOCAL, STATUS_NOT_READY,
                                                pack_counter, unpack_counter)

    assert pack_counter(STATUS_LOCAL, 15) == 0x4000000F
    assert pack_counter(STATUS_GLOBAL, 53) == 0x80000035
    assert pack_counter(STATUS_NOT_READY, 0) == 0
    for status in (0, 1, 2):
        for value in (0, 1, 2**30 - 1):
            assert unpack_counter(pack_counter(status, value)) == (status, value)
    with pytest.raises(ValueError):
        pack_counter(STATUS_LOCAL, 1 << 30)
    with pytest.raises(ValueError):
        pack_counter(3, 0)


def test_executor_ledger():
    from paper_2206_01784_b200 import Executor, ledger_as_row

    ex = Executor(workers=3)
    ex.ledger_record("histogram", "element_reads", 10)
    ex.ledger_record("partition", "element_reads", 40)
    ex.ledger_record("partition", "element_writes", 40)
    snap = ex.ledger_snapshot()
    assert snap.element_ops == 90 and snap.phase("partition").element_writes == 40
    assert ledger_as_row(snap)["element_ops"] == 90
    with pytest.raises(ValueError):
        ex.ledger_record("x", "bogus", 1)
    with pytest.raises(ValueError):
        Executor(workers=0)
    ex.ledger_reset()
    assert ex.ledger_snapshot().element_ops == 0


def test_product_never_imports_oracle():
    # the product package never imports, loads or links the test oracle
    # (oracle/, liboracle.so); "oracle" as the reference CLI's algo name and
    # the comparator API oracle_stable_sort are not the oracle package
    pkg = os.path.join(ROOT, "paper_2206_01784_b200")
    bad = re.compile(r"(^|\n)\s*(from\s+oracle\b|import\s+oracle\b)|liboracle|or_sort|oracle/")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                text = re.sub(r"#.*|//.*", "", open(os.path.join(dirpath, f)).read())
                assert not bad.search(text), f
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, %r); import paper_2206_01784_b200, paper_2206_01784_b200.cli, "
            "paper_2206_01784_b200.distributed; print(any(m == 'oracle' or m.startswith('oracle.') "
            "for m in sys.modules))" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.stdout.strip() == "False", out.stdout + out.stderr


def test_entropy_table():
    # test_keygen.py:17-24
    from paper_2206_01784_b200 import expected_entropy

    for q, want in {1: 1.0, 2: 0.811278, 3: 0.543564, 4: 0.33729, 8: 0.036875, 16: 0.000266}.items():
        assert expected_entropy(q) == pytest.approx(want, abs=5e-6)


def test_gather_rows_argument_errors():
    """os_gather_rows validates its arguments before touching the device."""
    from paper_2206_01784_b200 import _native

    L = _native.load()
    assert L.os_gather_rows(None, None, 3, None, 0, 16, None) == _native.OS_ERR_ARG
    assert L.os_gather_rows(None, None, 4, None, 10, 16, None) == _native.OS_ERR_ARG
    assert L.os_gather_rows(None, None, 8, None, 0, 16, None) == _native.OS_OK  # empty: no-op
