"""pytest plugin: run the reference's own test files against the drop-in.

`import onesweep` (and every `onesweep.<module>` the reference tests import:
keycodec, keygen, histogram, binning, baseline, lookback, executor, cli)
resolves to paper_2206_01784_b200 and its same-named modules, so the tests
exercise the device path unmodified.  The reference test files are not
committed: tools/stage_reference_suite.sh copies them from
/root/reference/pkg/tests into oracle/_ref/reference_tests/ (git-ignored, it
travels to the GPU box with the snapshot).  Tests that exercise the
reference's CPU thread pool or its mutable CounterMatrix -- the parts the CUDA
grid replaces -- are listed with a reason in
tests/reference_suite/xfail.txt and marked xfail(strict=False).

usage: python -m pytest -p onesweep_alias oracle/_ref/reference_tests
"""

from __future__ import annotations

import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

_MODULES = ("keycodec", "keygen", "histogram", "binning", "baseline", "lookback", "executor", "cli")


def _install_alias() -> None:
    pkg = importlib.import_module("paper_2206_01784_b200")
    sys.modules["onesweep"] = pkg
    for m in _MODULES:
        sys.modules[f"onesweep.{m}"] = importlib.import_module(f"paper_2206_01784_b200.{m}")


_install_alias()


def _xfail_table() -> dict[str, str]:
    table = {}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "xfail.txt")
    if os.path.exists(path):
        for line in open(path):
            line = line.split("#", 1)[0].strip()
            if line:
                nodeid, _, reason = line.partition(" ")
                table[nodeid] = reason.strip() or "out of scope"
    return table


def pytest_collection_modifyitems(config, items):
    import pytest

    table = _xfail_table()
    for item in items:
        name = f"{os.path.basename(item.fspath)}::{item.name}"
        base = name.split("[", 1)[0]
        reason = table.get(name) or table.get(base)
        if reason:
            item.add_marker(pytest.mark.xfail(reason=reason, strict=False))
