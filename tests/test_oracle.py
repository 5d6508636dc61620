"""Pins the CPU oracle (oracle/sstat_oracle.c) to the reference: golden vectors from the
reference's own tests and library, and bit-for-bit agreement with the reference library."""
from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest

from conftest import bits, unhex


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def gen_input(oracle, g):
    return oracle.generate(g["kind"], g["seed"], g["mu"], g["n_int"], 0, g["n"], g["p"])


def test_kats_single_row_and_identity(oracle, golden):
    for name in ("single_row", "orthogonal"):
        c = golden[name]
        n, s, S = oracle.accumulate_chunk(np.array(c["rows"]), c["p"])
        assert n == c["n"]
        assert np.array_equal(bits(s), bits(unhex(c["sums"])))
        assert np.array_equal(bits(S), bits(unhex(c["cross"])))
    # test_suffstats.cpp:45-52: S = [[1,2],[2,4]]
    assert list(unhex(golden["single_row"]["cross"])) == [1.0, 2.0, 4.0]


def test_kat_nonfinite_row_col(oracle, golden):
    c = golden["nonfinite_chunk"]
    rows = np.array([[1.0, 2.0], [3.0, np.inf]])
    res = oracle.accumulate_chunk(rows, 2, start_row=c["start_row"])
    assert res == ("nonfinite", c["error"]["row"], c["error"]["col"]) == ("nonfinite", 41, 1)


def test_table1_generator_and_accumulation_bit_exact(oracle, golden):
    c = golden["table1_seed21"]
    X = oracle.table1_chunk(21, 1, 10000)
    assert sha(X) == c["input_sha256"]
    n, s, S = oracle.accumulate_chunk(X, 11)
    assert n == 10000
    assert np.array_equal(bits(s), bits(unhex(c["sums"])))
    assert np.array_equal(bits(S), bits(unhex(c["cross"])))
    c32 = golden["table1_seed21_binary32"]
    _, s32, S32 = oracle.accumulate_chunk(X, 11, precision=1)
    assert np.array_equal(bits(S32), bits(unhex(c32["cross"])))
    assert np.array_equal(bits(s32), bits(unhex(c32["sums"])))


def test_dataset_fold_any_workers(oracle, golden):
    c = golden["table1_seed5_dataset"]
    X = oracle.table1_chunk(5, 1, 20000)
    assert sha(X) == c["input_sha256"]
    s0, c0 = oracle.plan_partitions(20000, 1024)
    for workers in (1, 2, 3, 8):
        n, s, S = oracle.run_reduction(X, 11, s0, c0, workers)
        assert n == 20000
        assert np.array_equal(bits(s), bits(unhex(c["sums"])))
        assert np.array_equal(bits(S), bits(unhex(c["cross"])))


def test_binary32_merge(oracle, golden):
    c = golden["binary32_merge"]
    a = oracle.accumulate_chunk(np.array([[16777216.0]]), 1, precision=1)
    b = oracle.accumulate_chunk(np.array([[1.0]]), 1, precision=1)
    assert oracle.merge(1, 1, a, b)[1][0] == float.fromhex(c["merged32"]) == 16777216.0
    a = oracle.accumulate_chunk(np.array([[16777216.0]]), 1)
    b = oracle.accumulate_chunk(np.array([[1.0]]), 1)
    assert oracle.merge(1, 0, a, b)[1][0] == float.fromhex(c["merged64"]) == 16777217.0


@pytest.mark.parametrize("name", ["c1_small", "c2_small", "c2_mu0", "ragged_p5", "p24", "p64", "wide_p80", "wide_p256"])
def test_generated_cases(oracle, golden, name):
    c = golden[name]
    g = c["gen"]
    X = gen_input(oracle, g)
    assert sha(X) == c["input_sha256"], "generator drifted from the pinned bytes"
    s0, c0 = oracle.plan_partitions(g["n"], g["chunk"])
    n, s, S = oracle.run_reduction(X, g["p"], s0, c0, workers=4)
    assert n == c["n"]
    assert np.array_equal(bits(s), bits(unhex(c["sums"])))
    if "cross" in c:
        assert np.array_equal(bits(S), bits(unhex(c["cross"])))
    else:
        assert sha(S) == c["cross_sha256"]


def test_generated_reduction_matches_in_memory(oracle):
    s0, c0 = oracle.plan_partitions(30000, 4096)
    X = oracle.generate(0, 9, 1.0, 2, 0, 30000, 16)
    a = oracle.run_reduction(X, 16, s0, c0, 3)
    b = oracle.generated_reduction(0, 9, 1.0, 2, 16, s0, c0, 5)
    assert a[0] == b[0]
    assert np.array_equal(bits(a[2]), bits(b[2]))


def test_dataset_nonfinite_lowest_range(oracle, golden):
    c = golden["dataset_nonfinite"]
    g = c["gen"]
    X = gen_input(oracle, g)
    for r, col, kind in c["poison"]:
        X[r, col] = np.inf if kind == "inf" else np.nan
    s0, c0 = oracle.plan_partitions(g["n"], g["chunk"])
    res = oracle.run_reduction(X, g["p"], s0, c0, 4)
    assert res[0] == "nonfinite"
    assert res[1] == c["error"]["range_index"] == 2
    assert (res[2], res[3]) == (3000, 5)
    assert c["error"]["msg"] == "range 2 failed: non-finite value at row 3000, column 5"


def test_plan_partitions(oracle, golden):
    for key, (starts, counts) in golden["plan_partitions"].items():
        n, k = eval(key)
        s, c = oracle.plan_partitions(n, k)
        assert list(map(int, s)) == starts and list(map(int, c)) == counts
    assert oracle.L.oracle_plan_partitions(10, 0, None, None) == 0
    assert oracle.L.oracle_plan_partitions(0, 5, None, None) == 0


def test_column_sum_kats(oracle, golden):
    for name, c in golden["column_sum"].items():
        v = c["values"]
        arr = (np.arange(1, int(v.split(":")[1]) + 1, dtype=np.float64) if isinstance(v, str) else unhex(v))
        s, k = oracle.plan_partitions(arr.size, c["chunk"])
        fs, exact, note_row = oracle.column_sum(arr.reshape(-1, 1), 1, 0, s, k)
        assert float(fs).hex() == c["float_sum"]
        assert (None if exact is None else str(exact)) == c["exact"]
        if exact is None:
            assert f"row {note_row}" in c["note"]


def test_comoments_pair(oracle, golden):
    c = golden["comoments_pair"]
    u = oracle.accumulate_comoments(np.array([[1.0, 5.0]]), 2)
    v = oracle.accumulate_comoments(np.array([[3.0, 1.0]]), 2)
    m = oracle.merge_comoments(2, u, v)
    assert m[0] == c["n"]
    assert np.array_equal(bits(m[1]), bits(unhex(c["mean"])))
    assert np.array_equal(bits(m[2]), bits(unhex(c["m2"])))


# ---- direct agreement with the reference library (random shapes, ragged chunks)
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_oracle_matches_reference_random(oracle, reference, seed, tmp_path):
    rng = np.random.default_rng(seed)
    p = int(rng.integers(1, 40))
    n = int(rng.integers(1, 5000))
    chunk = int(rng.integers(1, 2000))
    X = rng.normal(3.0, 2.0, size=(n, p))
    X[:, 0] = rng.integers(-50, 50, size=n)
    f = tmp_path / "x.bin"
    reference.write_binary(str(f), X, p)
    ref = reference.dataset_suffstats(str(f), p, chunk, 3)
    s, k = oracle.plan_partitions(n, chunk)
    got = oracle.run_reduction(X, p, s, k, 2)
    assert got[0] == ref[0]
    assert np.array_equal(bits(got[1]), bits(ref[1]))
    assert np.array_equal(bits(got[2]), bits(ref[2]))
    for prec in (0, 1):
        a = oracle.accumulate_chunk(X, p, 7, prec)
        b = reference.accumulate_chunk(X, p, 7, prec)
        assert np.array_equal(bits(a[2]), bits(b[2]))


def test_iid_generator_rowrng_matches_reference(oracle, reference):
    for idx in (1, 2, 1000, 123456789):
        assert np.array_equal(bits(oracle.iid_row(77, idx, 10, -1.0, 2.0)),
                              bits(reference.generate_row(1, 77, idx, iid_columns=10, lo=-1.0, hi=2.0)))
