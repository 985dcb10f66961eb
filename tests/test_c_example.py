"""The C ABI from a plain-C program (examples/sort_keys.c): builds against
include/onesweep_b200.h and the in-tree library with gcc alone (no Python,
no torch), and on the GPU sorts device-generated keys with their indices as
values and checks order, permutation and stability on the host."""

from __future__ import annotations

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2206_01784_b200", "_lib", "libonesweep_b200.so")
EXE = os.path.join(ROOT, "examples", "sort_keys")


def _build():
    if not os.path.exists(LIB):
        pytest.skip("library not built (run __graft_entry__.build())")
    if shutil.which("gcc") is None or not os.path.exists("/usr/local/cuda/include/cuda_runtime_api.h"):
        pytest.skip("gcc or CUDA headers missing")
    r = subprocess.run(["make", "-s", "-B", "-C", os.path.join(ROOT, "examples")],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    return EXE


def test_c_example_builds():
    assert os.access(_build(), os.X_OK)


@pytest.mark.gpu
@pytest.mark.parametrize("kt", ["u32", "u64", "i32", "i64", "f32", "f64"])
@pytest.mark.parametrize("values", [0, 1])
def test_c_example_runs(cuda, kt, values):
    exe = _build()
    r = subprocess.run([exe, "20", kt, str(values)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr


@pytest.mark.gpu
def test_c_example_c2_size(cuda):
    exe = _build()
    r = subprocess.run([exe, "28", "u32", "0"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr
