"""CPU-side checks of the product library: it builds, loads, exports every C-ABI symbol
declared in include/sstat_cuda.h, and its host helpers agree with the oracle."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, bits, gpu_available


def header_functions():
    src = open(os.path.join(ROOT, "include", "sstat_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(sstat_[a-z_0-9]+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2604_23826_b200 import _native as N

    lib = N.load()
    declared = header_functions()
    assert len(declared) >= 15
    assert sorted(N.EXPORTS) == declared
    nm = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True, check=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}\b", nm), name
        assert getattr(lib, name) is not None
    assert lib.sstat_cuda_abi_version() == 2


def test_library_is_sm100a():
    from paper_2604_23826_b200 import _native as N

    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", N.LIB_PATH], capture_output=True, text=True, check=True).stdout
    assert "DMMA" in sass  # FP64 tensor-pipe MMA in K1


def test_missing_library_fails_loudly(tmp_path):
    from paper_2604_23826_b200 import _native as N

    saved = N._lib
    N._lib = None
    try:
        with pytest.raises(N.NativeLibraryError):
            N.load(str(tmp_path / "nope.so"))
    finally:
        N._lib = saved


@pytest.mark.skipif(gpu_available(), reason="checks the no-device path")
def test_init_without_device_reports_cuda_error():
    from paper_2604_23826_b200 import DeviceError, Engine

    with pytest.raises(DeviceError):
        Engine(0)


def test_plan_partitions_matches_oracle(oracle):
    from paper_2604_23826_b200 import _native as N
    from paper_2604_23826_b200 import plan_partitions

    lib = N.load()
    for n, k in [(10, 4), (10, 10), (10000000, 1000000), (1, 1), (5000, 137), (10**10, 1 << 20)]:
        R = lib.sstat_plan_partitions(n, k, None, None)
        s = np.zeros(R, dtype=np.uint64)
        c = np.zeros(R, dtype=np.uint64)
        lib.sstat_plan_partitions(n, k, s.ctypes.data, c.ctypes.data)
        if n < 10**9:
            os_, oc = oracle.plan_partitions(n, k)
            assert np.array_equal(s, os_) and np.array_equal(c, oc)
            part = plan_partitions(n, k)
            assert [r.start_row for r in part.ranges] == list(map(int, s))
        assert int(c.sum()) == n
    assert lib.sstat_plan_partitions(0, 5, None, None) == 0
    assert lib.sstat_plan_partitions(5, 0, None, None) == 0
    with pytest.raises(ValueError):
        plan_partitions(10, 0)


def test_shard_ranges_contiguous_cover():
    from paper_2604_23826_b200 import shard_ranges

    for R in (1, 7, 96, 954, 9537):
        for W in (1, 2, 3, 4, 8):
            spans = [shard_ranges(R, q, W) for q in range(W)]
            assert spans[0][0] == 0 and spans[-1][1] == R
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and b >= a
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_ranges(10, 2, 2)


def test_merge_matches_oracle_and_reference_semantics(oracle):
    from paper_2604_23826_b200 import DatasetSchema, PrecisionMode, SchemaMismatchError, SuffStats, merge_suffstats

    rng = np.random.default_rng(5)
    X, Y = rng.normal(size=(100, 6)), rng.normal(size=(50, 6))
    for prec in (0, 1):
        a, b = oracle.accumulate_chunk(X, 6, 0, prec), oracle.accumulate_chunk(Y, 6, 100, prec)
        want = oracle.merge(6, prec, a, b)
        sch = DatasetSchema.generic(6)
        A = SuffStats(a[0], a[1], a[2], sch, PrecisionMode(prec))
        B = SuffStats(b[0], b[1], b[2], sch, PrecisionMode(prec))
        m = merge_suffstats(A, B)
        assert m.n == want[0] == 150
        assert np.array_equal(bits(m.cross), bits(want[2])) and np.array_equal(bits(m.sums), bits(want[1]))
        assert merge_suffstats(A, SuffStats.empty(sch, PrecisionMode(prec))) == A
    with pytest.raises(SchemaMismatchError):
        merge_suffstats(SuffStats.empty(DatasetSchema.table1()), SuffStats.empty(DatasetSchema.generic(11)))
    with pytest.raises(SchemaMismatchError):
        merge_suffstats(SuffStats.empty(DatasetSchema.table1()),
                        SuffStats.empty(DatasetSchema.table1(), PrecisionMode.Binary32Diagnostic))


def rank_layout(partials_per_rank, p, R, W):
    """Pack per-rank range partials into the all-gather layout (4-double header + lmax slots)."""
    E = p + p * (p + 1) // 2
    lmax = (R + W - 1) // W
    stride = 4 + lmax * E
    buf = np.full(W * stride, np.nan)
    for q, part in enumerate(partials_per_rank):
        buf[q * stride: q * stride + 4] = 0.0
        buf[q * stride + 4: q * stride + 4 + part.size] = part.reshape(-1)
    return buf, stride


@pytest.mark.parametrize("W", [1, 2, 3, 4, 8])
def test_host_fold_equals_reference_fold_for_any_world(oracle, W):
    """The fold code shared by K3b and sstat_fold_ranges_host, over the rank layout,
    equals the reference's ascending merge of per-range partials (reduce.hpp:142-145)."""
    from paper_2604_23826_b200 import _native as N
    from paper_2604_23826_b200 import shard_ranges

    lib = N.load()
    p, n, chunk = 7, 3000, 211
    X = oracle.generate(0, 4, 1.0, 2, 0, n, p)
    s, c = oracle.plan_partitions(n, chunk)
    R = len(s)
    parts = []
    for i in range(R):
        nn, ss, SS = oracle.accumulate_chunk(X[int(s[i]): int(s[i] + c[i])], p, int(s[i]))
        parts.append(np.concatenate([ss, SS]))
    per_rank = []
    for q in range(W):
        f, l = shard_ranges(R, q, W)
        per_rank.append(np.array(parts[f:l]))
    buf, stride = rank_layout(per_rank, p, R, W)
    E = p + p * (p + 1) // 2
    out = np.zeros(E)
    dp = ctypes.POINTER(ctypes.c_double)
    assert lib.sstat_fold_ranges_host(buf.ctypes.data_as(dp), stride, R, W, p, 0, 2, out.ctypes.data_as(dp)) == 0
    want = oracle.run_reduction(X, p, s, c, 1)
    assert np.array_equal(bits(out[:p]), bits(want[1]))
    assert np.array_equal(bits(out[p:]), bits(want[2]))


@pytest.mark.parametrize("W", [1, 2, 3, 8])
def test_host_fast_fold_is_the_32_lane_order(oracle, W):
    """The default-mode fold: lane q sums ranges q, q+32, ... from +0.0, then lanes 0..31 in
    order — the same bits for any rank layout."""
    from paper_2604_23826_b200 import _native as N
    from paper_2604_23826_b200 import shard_ranges

    lib = N.load()
    rng = np.random.default_rng(W)
    p, R = 5, 137
    E = p + p * (p + 1) // 2
    parts = rng.normal(size=(R, E)) * 10.0 ** rng.integers(-8, 8, size=(R, E))
    per_rank = [parts[shard_ranges(R, q, W)[0]:shard_ranges(R, q, W)[1]] for q in range(W)]
    buf, stride = rank_layout(per_rank, p, R, W)
    out = np.zeros(E)
    dp = ctypes.POINTER(ctypes.c_double)
    assert lib.sstat_fold_ranges_host(buf.ctypes.data_as(dp), stride, R, W, p, 0, 0, out.ctypes.data_as(dp)) == 0
    want = np.zeros(E)
    for e in range(E):
        t = 0.0
        for q in range(32):
            s = 0.0
            for r in range(q, R, 32):
                s += parts[r, e]
            t += s
        want[e] = t
    assert np.array_equal(bits(out), bits(want))


def test_fold_range_partials_resume_equals_reference(oracle):
    """fold_range_partials (the resume half of checkpoint/resume) over the reference's own
    per-range partials gives the reference's dataset result bit-for-bit in reference order,
    and rejects a partial set of the wrong size."""
    from paper_2604_23826_b200 import DatasetSchema, ReductionPlan, fold_range_partials, plan_partitions

    p, n, chunk = 6, 2500, 173
    X = oracle.generate(0, 9, 1.0, 2, 0, n, p)
    s, c = oracle.plan_partitions(n, chunk)
    parts = [np.concatenate(oracle.accumulate_chunk(X[int(a): int(a + b)], p, int(a))[1:]) for a, b in zip(s, c)]
    plan = ReductionPlan(plan_partitions(n, chunk))
    schema = DatasetSchema.generic(p, False)
    got = fold_range_partials(np.array(parts), schema, plan, flags=2)
    want = oracle.run_reduction(X, p, s, c, 1)
    assert got.n == n
    assert np.array_equal(bits(got.sums), bits(want[1])) and np.array_equal(bits(got.cross), bits(want[2]))
    with pytest.raises(ValueError):
        fold_range_partials(np.array(parts[:-1]), schema, plan)


def test_partition_arrays_follow_in_place_edits():
    """Partition's cached C-ABI arrays are keyed on the ranges' contents (a mutation counter on
    the list), so replacing a middle RowRange in place, appending, or reassigning the list is seen
    (keyed on (id, len, last) it reused stale arrays)."""
    from paper_2604_23826_b200 import RowRange, plan_partitions

    part = plan_partitions(100, 10)
    s0, c0 = part.arrays()
    assert list(s0[:3]) == [0, 10, 20]
    part.ranges[1] = RowRange(10, 5)
    s1, c1 = part.arrays()
    assert list(c1[:3]) == [10, 5, 10]
    part.ranges.append(RowRange(100, 7))
    assert part.arrays()[1][-1] == 7 and len(part.arrays()[0]) == 11
    part.ranges = [RowRange(0, 3)]
    assert list(part.arrays()[1]) == [3]
    a0 = part.addresses()
    assert part.addresses() == a0  # unchanged plan: the same cached arrays


def test_array_width_checked_against_schema():
    """An (n, 12) array under an 11-column schema is the reference's SchemaMismatchError wrapped in
    ReductionError for range 0 (check_chunk, suffstats.cpp:33-36), not a coverage error."""
    from paper_2604_23826_b200 import ReductionError, SchemaMismatchError
    from paper_2604_23826_b200.sstat import _check_width

    _check_width(np.zeros((5, 11)), 11)
    _check_width(np.zeros(44), 11)
    with pytest.raises(ReductionError) as e:
        _check_width(np.zeros((5, 12)), 11)
    assert e.value.range_index() == 0 and isinstance(e.value.cause, SchemaMismatchError)
    assert "chunk has 12 columns, schema has 11" in str(e.value)
    with pytest.raises(ReductionError):
        _check_width(np.zeros(45), 11)
