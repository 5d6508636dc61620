"""Seeded random cases for the rest of the API surface, against the oracle (oracle/sstat_oracle.c,
the reference restated) and across sources:
  * column_sum (reduce.cpp:32-88): the exact 128-bit sum (or the first non-integral row) equals
    the oracle's; the reference-order float sum bit for bit; the fast float sum to rounding;
  * co-moments (suffstats.cpp:107-159): the oracle's per-range accumulate + ascending merge to
    1e-12 (Cauchy-Schwarz normalised), the same bits from every source;
  * range_partials in random checkpoint pieces, folded on the host (fold_range_partials), equal
    dataset_suffstats bit for bit in both modes; reference-order partials equal the oracle's;
  * non-finite values: the reference's error — lowest failing range, first bad (row, col) in
    row-major order — from the HBM, pageable-host, file and device-group passes."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import bits, cs_err

pytestmark = pytest.mark.gpu

REFEXACT = 2


def case(seed):
    rng = np.random.default_rng(5000 + seed)
    p = int(rng.integers(1, 65)) if rng.random() < 0.7 else int(rng.integers(65, 200))
    n = int(min(2_000_000, 2e9 / (p * (p + 2))) * rng.random() ** 1.5) + int(rng.integers(2, 40))
    k = rng.random()
    chunk = int(rng.integers(1, 300)) if k < 0.2 else n if k < 0.35 else int(rng.integers(1, n + 1))
    if (n + chunk - 1) // chunk > 5_000:
        chunk = (n + 4_999) // 5_000
    n_int = int(rng.integers(0, min(p, 3) + 1))
    mu = float(rng.choice([0.0, 1.0, 1e3]))
    return rng, p, n, chunk, n_int, mu


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


def group_parts(D, plan, W):
    from paper_2604_23826_b200 import shard_ranges

    R = len(plan.partition.ranges)
    parts = []
    for i in range(W):
        f, l = shard_ranges(R, i, W)
        if f == l:
            parts.append(D[:0])
            continue
        r0 = plan.partition.ranges[f].start_row
        r1 = plan.partition.ranges[l - 1].start_row + plan.partition.ranges[l - 1].row_count
        parts.append(D[r0:r1])
    return parts


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_column_sum_comoments_partials(engine, oracle, tmp_path, seed):
    import torch

    from paper_2604_23826_b200 import DatasetSchema, ReductionPlan, fold_range_partials, plan_partitions

    rng, p, n, chunk, n_int, mu = case(seed)
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 0, 300 + seed, mu, n_int, 0, n, p)
    torch.cuda.synchronize()
    H = D.cpu().numpy()
    plan = ReductionPlan(plan_partitions(n, chunk))
    sc = DatasetSchema.generic(p, False)
    starts, counts = oracle.plan_partitions(n, chunk)
    R = len(starts)
    what = f"p={p} n={n} chunk={chunk} n_int={n_int} mu={mu}"
    path = str(tmp_path / "x.bin")
    sstatbin(path, H)

    # column_sum: an integer-valued column (when there is one) and a Gaussian one
    cols = sorted({int(rng.integers(0, n_int)) if n_int else 0, int(rng.integers(0, p))})
    for col in cols:
        f_ref, exact_ref, bad_row = oracle.column_sum(H, p, col, starts, counts)
        for flags in (0, REFEXACT):
            res = [engine.column_sum(src, col, plan, p=p, flags=flags) for src in (D, H, path)]
            for r in res[1:]:
                assert bits(r.float_sum) == bits(res[0].float_sum) and r.exact_sum == res[0].exact_sum, what
            r = res[0]
            assert r.exact_sum == exact_ref, (what, col)
            if exact_ref is None:
                assert r.exact_note is not None and f"row {bad_row};" in r.exact_note, (what, col, r.exact_note)
            if flags == REFEXACT:
                assert bits(r.float_sum) == bits(f_ref), (what, col)
            else:
                scale = max(float(np.sum(np.abs(H[:, col]))), 1.0)
                assert abs(r.float_sum - f_ref) <= 1e-13 * scale, (what, col)

    # co-moments against the oracle's per-range accumulate + ascending merge
    acc = None
    for s0, c0 in zip(starts, counts):
        part = oracle.accumulate_comoments(H[int(s0): int(s0 + c0)], p, int(s0))
        acc = part if acc is None else oracle.merge_comoments(p, acc, part)
    cms = [engine.comoments(src, sc, plan) for src in (D, H, path)]
    for cm in cms[1:]:
        assert np.array_equal(bits(cm.m2), bits(cms[0].m2)) and np.array_equal(bits(cm.mean), bits(cms[0].mean)), what
    cm = cms[0]
    assert cm.n == acc[0] == n
    sd = np.sqrt(np.maximum(acc[2][[j * p - j * (j - 1) // 2 for j in range(p)]], 0.0) / n)
    assert np.all(np.abs(cm.mean - acc[1]) <= 1e-12 * (np.abs(acc[1]) + sd + 1e-300)), what
    if n > 1:
        assert cs_err(cm.m2, acc[2], p) <= 1e-12, what

    # checkpoint pieces: range_partials over random cuts of [0, R), folded on the host
    cuts = sorted(set([0, R] + [int(x) for x in rng.integers(0, R + 1, size=min(R, 3))]))
    for flags in (0, REFEXACT):
        pieces = [engine.range_partials(D, sc, plan, a, b, flags=flags) for a, b in zip(cuts, cuts[1:]) if b > a]
        parts = np.concatenate(pieces)
        assert parts.shape[0] == R
        folded = fold_range_partials(parts, sc, plan, flags=flags)
        whole = engine.dataset_suffstats(D, sc, plan, flags=flags)
        assert folded.bit_equal(whole), (what, flags)
        if flags == REFEXACT:
            for i in sorted({0, R - 1, int(rng.integers(0, R))}):
                want = oracle.accumulate_chunk(H[int(starts[i]): int(starts[i] + counts[i])], p, int(starts[i]))
                E = p + p * (p + 1) // 2
                assert np.array_equal(bits(parts[i]), bits(np.concatenate([want[1], want[2]])[:E])), (what, i)
    os.remove(path)
    del D
    torch.cuda.empty_cache()


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_nonfinite_error(engine, oracle, tmp_path, seed):
    import torch

    from paper_2604_23826_b200 import DatasetSchema, Engine, NonFiniteError, ReductionError, ReductionPlan, plan_partitions

    rng, p, n, chunk, n_int, mu = case(100 + seed)
    n = max(n, 64)
    H = oracle.generate(0, 900 + seed, mu, n_int, 0, n, p)
    for _ in range(int(rng.integers(1, 4))):  # 1-3 bad values anywhere
        H[int(rng.integers(0, n)), int(rng.integers(0, p))] = [np.nan, np.inf, -np.inf][int(rng.integers(0, 3))]
    starts, counts = oracle.plan_partitions(n, chunk)
    want = oracle.run_reduction(H, p, starts, counts, workers=4)
    assert want[0] == "nonfinite"
    _, w_range, w_row, w_col = want
    plan = ReductionPlan(plan_partitions(n, chunk))
    sc = DatasetSchema.generic(p, False)
    D = torch.from_numpy(H).cuda()
    path = str(tmp_path / "x.bin")
    sstatbin(path, H)
    g = Engine(devices=[0, 0, 0])
    try:
        for name, call in (("hbm", lambda f: engine.dataset_suffstats(D, sc, plan, flags=f)),
                           ("pageable", lambda f: engine.dataset_suffstats(H, sc, plan, flags=f)),
                           ("file", lambda f: engine.dataset_suffstats(path, sc, plan, flags=f)),
                           ("group", lambda f: g.dataset_suffstats(group_parts(D, plan, 3), sc, plan, flags=f))):
            for flags in (0, REFEXACT):
                with pytest.raises(ReductionError) as ei:
                    call(flags)
                e = ei.value
                assert e.range_index() == w_range, (name, flags, p, n, chunk)
                assert isinstance(e.cause, NonFiniteError)
                assert (e.cause.row(), e.cause.column()) == (w_row, w_col), (name, flags)
        # the engine is usable afterwards: a clean pass over finite rows
        Hc = np.nan_to_num(H, nan=0.0, posinf=0.0, neginf=0.0)
        assert engine.dataset_suffstats(Hc, sc, plan).n == n
    finally:
        g.close()
    os.remove(path)


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_chunks_readers_and_binary32(engine, oracle, seed):
    """accumulate_chunk on host and device chunks at random start rows (reference order: the
    oracle's bits; fast: within the bars), a RowReader source equal to the array source, and
    Binary32Diagnostic (the reference's float accumulation) bit-identical to the oracle."""
    import ctypes

    import torch

    from paper_2604_23826_b200 import (Chunk, DatasetSchema, PrecisionMode, ReductionPlan, RowReader,
                                       plan_partitions)

    rng, p, n, chunk, n_int, mu = case(200 + seed)
    H = oracle.generate(0, 1200 + seed, mu, n_int, 0, n, p)
    D = torch.from_numpy(H).cuda()
    sc = DatasetSchema.generic(p, False)
    what = f"p={p} n={n} chunk={chunk}"
    start = int(rng.integers(0, 1 << 40))
    want = oracle.accumulate_chunk(H, p, start)
    for vals in (H, D):
        exact = engine.accumulate_chunk(Chunk(start, n, p, vals), sc, flags=REFEXACT)
        assert exact.n == n and np.array_equal(bits(exact.cross), bits(want[2])), what
        assert np.array_equal(bits(exact.sums), bits(want[1])), what
        fast = engine.accumulate_chunk(Chunk(start, n, p, vals), sc)
        assert cs_err(fast.cross, want[2], p) <= 1e-12, what

    plan = ReductionPlan(plan_partitions(n, chunk))
    Hp = torch.from_numpy(H).pin_memory()

    def point(row, k, scratch):
        return Hp.data_ptr() + row * p * 8

    def fill(row, k, scratch):
        ctypes.memmove(scratch, H[row:row + k].ctypes.data, k * p * 8)
        return scratch

    base = engine.dataset_suffstats(D, sc, plan)
    for fn in (point, fill):
        assert engine.dataset_suffstats(RowReader(fn, n), sc, plan).bit_equal(base), (what, fn.__name__)

    starts, counts = oracle.plan_partitions(n, chunk)
    want32 = oracle.run_reduction(H, p, starts, counts, workers=4, precision=1)
    plan32 = ReductionPlan(plan_partitions(n, chunk), 1, PrecisionMode(1))
    for src in (D, H):
        got32 = engine.dataset_suffstats(src, sc, plan32)
        assert np.array_equal(bits(got32.sums), bits(want32[1])), what
        assert np.array_equal(bits(got32.cross), bits(want32[2])), what


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_groups_every_call(engine, seed):
    """Device groups of 1-6 members (more members than ranges included) on random plans: every
    call — dataset in both modes, co-moments, column_sum, range_partials — gives the single-device
    bits, from per-member CUDA shards and from one shared host array."""
    import torch

    from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions

    rng, p, n, chunk, n_int, mu = case(400 + seed)
    W = int(rng.integers(1, 7))
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 0, 500 + seed, mu, n_int, 0, n, p)
    torch.cuda.synchronize()
    H = D.cpu().numpy()
    plan = ReductionPlan(plan_partitions(n, chunk))
    sc = DatasetSchema.generic(p, False)
    R = len(plan.partition.ranges)
    what = f"W={W} p={p} n={n} R={R}"
    g = Engine(devices=[0] * W)
    try:
        parts = group_parts(D, plan, W)
        for flags in (0, REFEXACT):
            want = engine.dataset_suffstats(D, sc, plan, flags=flags)
            assert g.dataset_suffstats(parts, sc, plan, flags=flags).bit_equal(want), (what, flags)
            assert g.dataset_suffstats(H, sc, plan, flags=flags).bit_equal(want), (what, flags, "host")
        a, b = engine.comoments(D, sc, plan), g.comoments(parts, sc, plan)
        assert np.array_equal(bits(a.m2), bits(b.m2)) and np.array_equal(bits(a.mean), bits(b.mean)), what
        col = int(rng.integers(0, p))
        ca, cb = engine.column_sum(D, col, plan, p=p), g.column_sum(parts, col, plan, p=p)
        assert bits(ca.float_sum) == bits(cb.float_sum) and ca.exact_sum == cb.exact_sum, what
    finally:
        g.close()
