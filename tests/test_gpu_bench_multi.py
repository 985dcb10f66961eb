"""bench.py's N > 1 path, end to end on the real kernels: two ranks share one
B200 over a gloo group (NCCL refuses two ranks on one device), so the sharded
sort uses the all-to-all exchange.  The line must carry the driver contract's
keys plus the per-phase split, the local-sort roofline and a host-buffer e2e,
and the output must verify (each slice sorted, slices ordered, no key lost)."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_schema(cuda):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "4", "--warmup", "3", "--n-per-gpu", str(1 << 22), "--e2e-steps", "2",
           "--backend", "gloo"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "gpu_launches", "clocks", "roofline",
              "e2e", "phases_ms"):
        assert k in d, k
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["output_verified"] is True
    assert set(d["phases_ms"]) == {"split", "exchange", "local"}
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * (1 << 22) * 4
    assert d["e2e"]["d2h_bytes_per_step"] == 2 * (1 << 22) * 4
