"""GPU checks of the passes next to the path:
column_sum (reference src/reduce.cpp:32-88) and centered co-moments
(src/suffstats.cpp:107-159), against the reference's own known answers and library."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import bits, unhex

pytestmark = pytest.mark.gpu


def plan(n, chunk, precision=0):
    from paper_2604_23826_b200 import PrecisionMode, ReductionPlan, plan_partitions

    return ReductionPlan(plan_partitions(n, chunk), 1, PrecisionMode(precision))


def to_dev(X):
    import torch

    return torch.from_numpy(np.ascontiguousarray(X)).cuda()


def schema(p):
    from paper_2604_23826_b200 import DatasetSchema

    return DatasetSchema.generic(p, False)


# ------------------------------------------------------------------ column_sum
@pytest.mark.parametrize("flags", [0, 2])
def test_column_sum_kats(engine, golden, reference, tmp_path, flags):
    """test_reduce.cpp:106-168 known answers, through every source kind."""
    for name, c in golden["column_sum"].items():
        v = c["values"]
        arr = (np.arange(1, int(v.split(":")[1]) + 1, dtype=np.float64) if isinstance(v, str) else unhex(v))
        X = arr.reshape(-1, 1)
        f = tmp_path / f"{name}.bin"
        reference.write_binary(str(f), X, 1)
        for src in (X, to_dev(X), str(f)):
            r = engine.column_sum(src, 0, plan(arr.size, c["chunk"]), p=1, flags=flags)
            assert (None if r.exact_sum is None else str(r.exact_sum)) == c["exact"], name
            assert r.float_matches_exact == c["float_matches"], name
            if flags == 2 or c["exact"] is not None and abs(int(c["exact"])) < 2**53:
                assert float(r.float_sum).hex() == c["float_sum"], name
            if c["exact"] is None:
                assert r.exact_note is not None and r.exact_note in c["note"], (r.exact_note, c["note"])
    with pytest.raises(IndexError):
        engine.column_sum(np.zeros((5, 1)), 1, plan(5, 5), p=1)


def test_column_sum_identifier_checks(engine, oracle):
    """The paper's first validation: sum of the identifier column = n(n+1)/2,
    at C1 size and past 2^63 (exact 128-bit path)."""
    import torch

    n, p = 1_000_000, 9
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 1, 42, 1.0, 0, 0, n, p)
    r = engine.column_sum(D, 0, plan(n, 1 << 20))
    assert r.exact_sum == n * (n + 1) // 2 and r.float_matches_exact
    # Gaussian column: not integral, the note names the first non-integral row (row 0)
    r = engine.column_sum(D, 3, plan(n, 1 << 20))
    assert r.exact_sum is None and "row 0" in r.exact_note
    # values near 2^62: the exact sum needs more than 64 bits
    big = np.full((1000, 1), float(2**62))
    r = engine.column_sum(to_dev(big), 0, plan(1000, 64), p=1)
    assert r.exact_sum == 1000 * 2**62
    assert r.float_matches_exact  # 1000 * 2^62 is exactly representable
    # chunk-size invariance of the exact sum (test_reduce.cpp:160-168) at 1e8 rows
    n = 100_000_000
    ids = torch.arange(1, n + 1, dtype=torch.float64, device="cuda").reshape(-1, 1)
    a = engine.column_sum(ids, 0, plan(n, 1 << 20), p=1)
    b = engine.column_sum(ids, 0, plan(n, 777_777), p=1)
    assert a.exact_sum == b.exact_sum == n * (n + 1) // 2
    assert a.float_matches_exact


def test_column_sum_binary32_matches_reference(engine, reference, tmp_path):
    rng = np.random.default_rng(3)
    X = rng.normal(100.0, 3.0, size=(20000, 3))
    f = tmp_path / "x.bin"
    reference.write_binary(str(f), X, 3)
    ref = reference.column_sum(str(f), 1, 1024, 2, precision=1)
    got = engine.column_sum(str(f), 1, plan(20000, 1024, precision=1), p=3)
    assert got.float_sum == ref[0]
    ref64 = reference.column_sum(str(f), 1, 1024, 2, precision=0)
    got64 = engine.column_sum(to_dev(X), 1, plan(20000, 1024), p=3, flags=2)
    assert float(got64.float_sum).hex() == float(ref64[0]).hex()


# ------------------------------------------------------------------ co-moments
def test_comoments_pair_kat(engine, golden):
    """test_suffstats.cpp:159-172: two single rows, the pairwise algebra."""
    c = golden["comoments_pair"]
    X = np.array([[1.0, 5.0], [3.0, 1.0]])
    cm = engine.comoments(X, schema(2), plan(2, 1))
    assert cm.n == c["n"] == 2
    assert np.allclose(cm.mean, unhex(c["mean"]), rtol=1e-15, atol=0)
    assert np.allclose(cm.m2, unhex(c["m2"]), rtol=1e-14, atol=0)
    assert list(cm.m2) == [2.0, -4.0, 8.0]


def test_comoments_identifier_variance(engine):
    """test_suffstats.cpp:174-192: variance of 1..n is n(n+1)/12 within 1e-12 at n = 1e6."""
    import torch

    n = 1_000_000
    ids = torch.arange(1, n + 1, dtype=torch.float64, device="cuda").reshape(-1, 1)
    cm = engine.comoments(ids, schema(1), plan(n, 65536))
    expected = n * (n + 1) / 12.0
    assert abs(cm.m2[0] / (n - 1) - expected) <= 1e-12 * expected
    assert cm.mean[0] == (n + 1) / 2


def test_comoments_vs_reference_and_two_pass(engine, oracle, reference):
    """Table1 seed 31 (test_suffstats.cpp:194-205): against the reference's chunk two-pass
    co-moments, and multi-range merges against an extended-precision two-pass."""
    X = oracle.table1_chunk(31, 1, 10000)
    n, ref_mean, ref_m2 = reference.accumulate_comoments(X, 11)
    cm = engine.comoments(to_dev(X), schema(11), plan(10000, 10000))
    assert cm.n == n
    iu = np.triu_indices(11)
    diag = ref_m2[[j * 11 - j * (j - 1) // 2 for j in range(11)]]
    scale = np.sqrt(np.abs(diag[iu[0]] * diag[iu[1]]))
    assert np.max(np.abs(cm.m2 - ref_m2) / scale) <= 1e-12
    assert np.max(np.abs(cm.mean - ref_mean) / np.abs(ref_mean)) <= 1e-13
    # many ranges + the pairwise merge, mu = 1000 data (where raw moments cancel)
    rng = np.random.default_rng(9)
    Y = 1000.0 + rng.normal(size=(200_003, 6)) @ np.triu(np.ones((6, 6)))
    L = Y.astype(np.longdouble)
    mu = L.mean(axis=0)
    C = (L - mu).T @ (L - mu)
    cm = engine.comoments(to_dev(Y), schema(6), plan(len(Y), 4099))
    M2 = np.zeros((6, 6))
    M2[np.triu_indices(6)] = cm.m2
    M2 = M2 + np.triu(M2, 1).T
    d = np.sqrt(np.outer(np.diag(C), np.diag(C))).astype(np.float64)
    assert np.max(np.abs(M2 - C.astype(np.float64)) / d) <= 1e-12
    assert np.max(np.abs(cm.mean - mu.astype(np.float64))) <= 1e-12 * 1000


@pytest.mark.parametrize("p", [80, 256])
def test_comoments_wide_p(engine, p):
    """Co-moments through K2 (p > 64): mean 50 data over ragged ranges against an 80-bit
    two-pass (CS-normalised 1e-12), and the reference's merge order is irrelevant to the bar."""
    rng = np.random.default_rng(p)
    n = 60_001
    Y = 50.0 + rng.normal(size=(n, p))
    L = Y.astype(np.longdouble)
    mu = L.mean(axis=0)
    C = ((L - mu).T @ (L - mu)).astype(np.float64)
    cm = engine.comoments(to_dev(Y), schema(p), plan(n, 7919))
    assert cm.n == n
    iu = np.triu_indices(p)
    scale = np.sqrt(np.abs(np.diag(C)[iu[0]] * np.diag(C)[iu[1]]))
    assert np.max(np.abs(cm.m2 - C[iu]) / scale) <= 1e-12
    assert np.max(np.abs(cm.mean - mu.astype(np.float64)) / np.abs(mu.astype(np.float64))) <= 1e-14
