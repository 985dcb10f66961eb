"""CLI (paper_2206_01784_b200/cli.py): the reference CLI's contract
(cli.py:1-339, tests at test_cli.py:1-252) -- round trips through the device
sorts, verification diagnostics, exit codes and the bench CSV."""

from __future__ import annotations

import csv
import io
from contextlib import redirect_stderr, redirect_stdout

import numpy as np
import pytest


def cli(*argv):
    from paper_2206_01784_b200.cli import main

    out, err = io.StringIO(), io.StringIO()
    with redirect_stdout(out), redirect_stderr(err):
        code = main(list(argv))
    return code, out.getvalue(), err.getvalue()


# -- host-only behaviour (no device work happens before these fail) -------------


def test_malformed_file_size_is_a_data_error(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"\x01\x02\x03")
    code, _, err = cli("sort", "--in", str(bad), "--out", str(tmp_path / "o.bin"))
    assert code == 1 and "malformed" in err


def test_missing_input_names_the_path(tmp_path):
    code, _, err = cli("sort", "--in", str(tmp_path / "nope.bin"), "--out", str(tmp_path / "o.bin"))
    assert code == 1 and "nope.bin" in err


def test_usage_errors_exit_2(tmp_path):
    with pytest.raises(SystemExit) as e:
        cli("sort", "--in", "x", "--out", "y", "--key-type", "u128")
    assert e.value.code == 2
    raw = tmp_path / "in.bin"
    np.arange(4, dtype="<u4").tofile(raw)
    with pytest.raises(SystemExit) as e:
        cli("sort", "--in", str(raw), "--out", str(tmp_path / "o.bin"), "--key-type", "u64", "--bits", "32")
    assert e.value.code == 2


def test_verify_count_mismatch(tmp_path):
    a, b = tmp_path / "a.bin", tmp_path / "b.bin"
    np.arange(10, dtype="<u4").tofile(a)
    np.arange(8, dtype="<u4").tofile(b)
    code, _, err = cli("verify", "--in", str(a), "--sorted", str(b))
    assert code == 1 and "mismatch" in err


def test_bad_sizes_is_a_data_error():
    code, _, err = cli("bench", "--sizes", "nonsense")
    assert code == 1 and "--sizes" in err


# -- device round trips ----------------------------------------------------------


@pytest.mark.gpu
def test_gen_empty_and_deterministic(cuda, tmp_path):
    from paper_2206_01784_b200 import KeyGenSpec, empirical_bit_entropy, generate_keys

    e = tmp_path / "e.bin"
    assert cli("gen", "--n", "0", "--out", str(e))[0] == 0 and e.stat().st_size == 0
    a, b = tmp_path / "a.bin", tmp_path / "b.bin"
    for p in (a, b):
        assert cli("gen", "--n", str(1 << 16), "--q", "1", "--seed", "3", "--out", str(p))[0] == 0
    assert a.read_bytes() == b.read_bytes() and a.stat().st_size == 4 << 16
    assert abs(empirical_bit_entropy(np.fromfile(a, dtype="<u4")) - 1.0) < 0.01
    c = tmp_path / "c.bin"
    cli("gen", "--n", "1000", "--q", "4", "--seed", "9", "--out", str(c))
    assert np.array_equal(np.fromfile(c, dtype="<u4"), generate_keys(KeyGenSpec(q=4, seed=9, n=1000)))


@pytest.mark.gpu
@pytest.mark.parametrize("key_type", ["u32", "i32", "f32", "u64", "i64", "f64"])
@pytest.mark.parametrize("algo", ["onesweep", "rts", "oracle"])
def test_gen_sort_verify_roundtrip(cuda, oracle, tmp_path, key_type, algo):
    bits = "64" if key_type.endswith("64") else "32"
    raw, out = tmp_path / "in.bin", tmp_path / "out.bin"
    assert cli("gen", "--n", "5000", "--q", "2", "--seed", "11", "--bits", bits, "--out", str(raw))[0] == 0
    assert cli("sort", "--in", str(raw), "--out", str(out), "--key-type", key_type, "--algo", algo)[0] == 0
    code, msg, err = cli("verify", "--in", str(raw), "--sorted", str(out), "--key-type", key_type)
    assert code == 0 and "ok" in msg, err
    # and against the C oracle pinned to the reference
    w = "<u8" if bits == "64" else "<u4"
    want = oracle.sort(np.fromfile(raw, dtype=w).view(np.dtype(KEY_DT[key_type])))
    assert np.array_equal(np.fromfile(out, dtype=w), want.view(w))


KEY_DT = {"u32": "<u4", "i32": "<i4", "f32": "<f4", "u64": "<u8", "i64": "<i8", "f64": "<f8"}


@pytest.mark.gpu
def test_sort_idempotent_and_algorithms_agree(cuda, tmp_path):
    raw = tmp_path / "in.bin"
    cli("gen", "--n", "4000", "--q", "3", "--seed", "8", "--out", str(raw))
    blobs = []
    for algo in ("onesweep", "rts", "oracle"):
        o = tmp_path / f"{algo}.bin"
        assert cli("sort", "--in", str(raw), "--out", str(o), "--algo", algo, "--d", "6")[0] == 0
        blobs.append(o.read_bytes())
    assert blobs[0] == blobs[1] == blobs[2]
    twice = tmp_path / "twice.bin"
    cli("sort", "--in", str(tmp_path / "onesweep.bin"), "--out", str(twice))
    assert twice.read_bytes() == blobs[0]
    for w in ("1", "8"):  # worker counts are accepted and change nothing
        o = tmp_path / f"w{w}.bin"
        assert cli("sort", "--in", str(raw), "--out", str(o), "--workers", w, "--tile", "512")[0] == 0
        assert o.read_bytes() == blobs[0]


@pytest.mark.gpu
def test_values_and_verify_diagnostics(cuda, tmp_path):
    rng = np.random.default_rng(5)
    rec = np.empty((2000, 2), dtype="<u4")
    rec[:, 0] = rng.integers(0, 64, size=2000)
    rec[:, 1] = np.arange(2000)
    raw, out = tmp_path / "kv.bin", tmp_path / "kv-sorted.bin"
    rec.tofile(raw)
    assert cli("sort", "--in", str(raw), "--out", str(out), "--values", "--bits", "32")[0] == 0
    assert cli("verify", "--in", str(raw), "--sorted", str(out), "--values", "--bits", "32")[0] == 0
    # a swapped key pair names its index
    k_in, k_out = tmp_path / "k.bin", tmp_path / "k-sorted.bin"
    cli("gen", "--n", "1000", "--q", "1", "--seed", "6", "--out", str(k_in))
    cli("sort", "--in", str(k_in), "--out", str(k_out))
    d = np.fromfile(k_out, dtype="<u4")
    d[100], d[101] = d[101].copy(), d[100].copy()
    d.tofile(k_out)
    code, _, err = cli("verify", "--in", str(k_in), "--sorted", str(k_out))
    assert code == 1 and "index 100" in err
    # equal keys with the payload order inverted: a stability violation
    good = np.array([[7, 0], [7, 1], [7, 2], [7, 3]], dtype="<u4")
    bad = good.copy()
    bad[:, 1] = good[::-1, 1]
    good.tofile(tmp_path / "g.bin")
    bad.tofile(tmp_path / "b.bin")
    code, _, err = cli("verify", "--in", str(tmp_path / "g.bin"), "--sorted", str(tmp_path / "b.bin"),
                       "--values", "--bits", "32")
    assert code == 1 and "stability" in err


@pytest.mark.gpu
def test_bench_csv_rows_and_traffic(cuda, tmp_path):
    from paper_2206_01784_b200.cli import CSV_FIELDS

    p = tmp_path / "bench.csv"
    code, _, err = cli("bench", "--sizes", "10:11:2", "--q", "1,4", "--d", "8", "--algos", "onesweep,rts",
                       "--trials", "2", "--csv", str(p), "--seed", "1")
    assert code == 0, err
    with open(p, newline="") as fh:
        reader = csv.DictReader(fh)
        assert reader.fieldnames == CSV_FIELDS
        rows = list(reader)
    assert len(rows) == 16  # 2 sizes x 2 q x 1 d x 2 algos x 2 trials
    for r in rows:
        n, ops = int(r["n"]), int(r["element_ops"])
        if r["algo"] == "onesweep":
            assert ops == 9 * n and float(r["traffic_ratio"]) == pytest.approx(1.0)
        else:
            assert ops == 12 * n and float(r["traffic_ratio"]) == pytest.approx(1.3333, abs=1e-4)
        assert float(r["keys_per_sec"]) > 0 and r["trial"] in ("1", "2")


@pytest.mark.gpu
def test_bench_d_sweep_is_2p_plus_1(cuda, tmp_path):
    p = tmp_path / "sweep.csv"
    assert cli("bench", "--sizes", "10:10:1", "--q", "1", "--d", "5,6,7,8,9,11,16", "--algos", "onesweep",
               "--trials", "1", "--csv", str(p))[0] == 0
    with open(p, newline="") as fh:
        rows = list(csv.DictReader(fh))
    assert sorted({r["d"] for r in rows}, key=int) == ["5", "6", "7", "8", "9", "11", "16"]
    for r in rows:
        passes = -(-32 // int(r["d"]))
        assert int(r["element_ops"]) == (2 * passes + 1) * int(r["n"])
