"""Seeded random plans across every kernel family and tile-height rule: widths 1-300, row counts
from a few rows to a few million, chunk sizes from a handful of rows to the whole matrix (many
short ranges, ranges shorter than a tile, one range), integer-valued and Gaussian columns with
small and large means.  Per case:
  * the fast pass from HBM equals, bit for bit, the same pass from pinned and pageable host
    memory, from an SSTATBIN file (with the default and a random staging ring and feeder thread
    count) and from a two-member device group (one fixed function of the rows and the plan,
    whatever the source, staging or GPU count);
  * it agrees with the oracle's reference-order reduction (reduce.hpp:70-146 restated,
    oracle/sstat_oracle.c) to the Cauchy-Schwarz-normalised 1e-12 bar, integer-valued columns
    exactly;
  * the reference-order mode (SSTAT_FLAG_REFEXACT) equals the oracle bit for bit."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import bits, cs_err

pytestmark = pytest.mark.gpu

REFEXACT = 2


def case(seed):
    rng = np.random.default_rng(1000 + seed)
    u = rng.random()
    p = int(rng.integers(1, 65)) if u < 0.6 else int(rng.integers(65, 141)) if u < 0.85 else int(rng.integers(141, 301))
    budget = 4e9 / (p * (p + 2))  # oracle work (8 threads): about a second
    n = int(min(8_000_000, budget) * rng.random() ** 1.5) + int(rng.integers(1, 50))
    k = rng.random()
    chunk = (int(rng.integers(1, 200)) if k < 0.15 else n if k < 0.3 else int(rng.integers(1, n + 1)) if k < 0.7
             else 1 << int(rng.integers(8, 21)))
    n_int = int(rng.integers(0, min(p, 3) + 1))
    mu = float(rng.choice([0.0, 1.0, 1e3]))
    return p, n, max(1, chunk), n_int, mu


def sstatbin(path, H):
    n, p = H.shape
    hdr = bytearray(64)
    hdr[0:8] = b"SSTATBIN"
    hdr[8:12] = (1).to_bytes(4, "little")
    hdr[12:20] = int(n).to_bytes(8, "little")
    hdr[20:24] = int(p).to_bytes(4, "little")
    with open(path, "wb") as f:
        f.write(hdr)
        H.tofile(f)


@pytest.mark.parametrize("seed", range(48))
def test_fuzz_sources_groups_and_oracle(engine, oracle, tmp_path, seed):
    import torch

    from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions, shard_ranges

    p, n, chunk, n_int, mu = case(seed)
    if (n + chunk - 1) // chunk > 20_000:  # keep the plan arrays (and the oracle loop) small
        chunk = (n + 19_999) // 20_000
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 0, 77 + seed, mu, n_int, 0, n, p)
    torch.cuda.synchronize()
    H = D.cpu().numpy()
    plan = ReductionPlan(plan_partitions(n, chunk))
    sc = DatasetSchema.generic(p, False)
    what = f"p={p} n={n} chunk={chunk} n_int={n_int} mu={mu}"

    got = engine.dataset_suffstats(D, sc, plan)
    P = torch.empty((n, p), dtype=torch.float64, pin_memory=True)
    P.copy_(D)
    assert engine.dataset_suffstats(P, sc, plan).bit_equal(got), what + " pinned"
    assert engine.dataset_suffstats(H, sc, plan).bit_equal(got), what + " pageable"
    path = str(tmp_path / "x.bin")
    sstatbin(path, H)
    assert engine.dataset_suffstats(path, sc, plan).bit_equal(got), what + " file"
    # a second engine with a random staging ring (slots grow to the largest unit when smaller)
    rng = np.random.default_rng(seed)
    e2 = Engine(0)
    try:
        e2.set_staging(int(rng.integers(2, 6)), int(rng.integers(1 << 20, 64 << 20)))  # >= 1 MiB
        e2.set_host_threads(int(rng.integers(1, 9)))
        for src in (P, H, path):
            assert e2.dataset_suffstats(src, sc, plan).bit_equal(got), what + " staging"
    finally:
        e2.close()
    R = len(plan.partition.ranges)
    g = Engine(devices=[0, 0])
    try:
        parts = []
        for i in range(2):
            f, l = shard_ranges(R, i, 2)
            if f == l:
                parts.append(D[:0])
                continue
            r0 = plan.partition.ranges[f].start_row
            r1 = plan.partition.ranges[l - 1].start_row + plan.partition.ranges[l - 1].row_count
            parts.append(D[r0:r1])
        assert g.dataset_suffstats(parts, sc, plan).bit_equal(got), what + " group"
    finally:
        g.close()

    starts, counts = oracle.plan_partitions(n, chunk)
    want = oracle.run_reduction(H, p, starts, counts, workers=8)
    assert got.n == want[0] == n
    assert cs_err(got.cross, want[2], p) <= 1e-12, what
    scale = np.maximum(np.abs(want[1]), np.sqrt(np.abs(want[2][[j * p - j * (j - 1) // 2 for j in range(p)]]) * n))
    scale[scale == 0] = 1.0
    assert np.max(np.abs(got.sums - want[1]) / scale) <= 1e-12, what
    if n_int:  # integer-valued columns: their sums and products are exact (all < 2^53)
        assert np.array_equal(got.sums[:n_int], want[1][:n_int]), what
        idx = [j * p - j * (j - 1) // 2 + (k - j) for j in range(n_int) for k in range(j, n_int)]
        assert np.array_equal(got.cross[idx], want[2][idx]), what

    exact = engine.dataset_suffstats(D, sc, plan, flags=REFEXACT)
    assert np.array_equal(bits(exact.sums), bits(want[1])) and np.array_equal(bits(exact.cross), bits(want[2])), what
    del D, P
    os.remove(path)
    torch.cuda.empty_cache()
