"""GPU tests of the device group (sstat_cuda_init_devices: one process driving G devices), the
cross-rank failure path, the reader source, stream ordering and reference-order streaming in
pieces.

One B200 serves every case: a group that lists device 0 W times runs W members — W rank
buffers, the peer-copy exchange into member 0 and the device range fold (K3b) over a W-rank
gathered layout — exactly the multi-GPU path except for the transport, and it must give the
single-device bits (the multi-GPU north star: results bit-identical for any GPU count).
"""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

from conftest import bits, cs_err

pytestmark = pytest.mark.gpu


def torch_mod():
    import torch

    return torch


def schema(p):
    from paper_2604_23826_b200 import DatasetSchema

    return DatasetSchema.generic(p, False)


def plan(n, chunk, precision=0):
    from paper_2604_23826_b200 import PrecisionMode, ReductionPlan, plan_partitions

    return ReductionPlan(plan_partitions(n, chunk), 1, PrecisionMode(precision))


def shards(D, pl, W):
    """Member i's contiguous shard of the plan's ranges (shard_ranges), as its own tensor."""
    from paper_2604_23826_b200 import shard_ranges

    R = len(pl.partition.ranges)
    out = []
    for i in range(W):
        f, l = shard_ranges(R, i, W)
        if f == l:
            out.append(D[:0].contiguous())
            continue
        r0 = pl.partition.ranges[f].start_row
        r1 = pl.partition.ranges[l - 1].start_row + pl.partition.ranges[l - 1].row_count
        out.append(D[r0:r1].contiguous())
    return out


def gen(engine, n, p, kind=0, seed=42):
    torch = torch_mod()
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, kind, seed, 1.0, 2 if kind == 0 else 0, 0, n, p)
    return D


def test_group_of_one_is_the_device_context(engine, tmp_path):
    """sstat_cuda_init_devices(1, {0}) gives the single-device bits for every call shape."""
    from paper_2604_23826_b200 import Engine

    n, p, chunk = 250_003, 16, 8191
    D = gen(engine, n, p)
    pl = plan(n, chunk)
    g = Engine(devices=[0])
    assert g.n_devices == 1
    for flags in (0, 2):
        want = engine.dataset_suffstats(D, schema(p), pl, flags=flags)
        assert g.dataset_suffstats([D], schema(p), pl, flags=flags).bit_equal(want)
        assert g.dataset_suffstats(D.cpu().numpy(), schema(p), pl, flags=flags).bit_equal(want)
    cm_a, cm_b = engine.comoments(D, schema(p), pl), g.comoments([D], schema(p), pl)
    assert np.array_equal(bits(cm_a.m2), bits(cm_b.m2)) and np.array_equal(bits(cm_a.mean), bits(cm_b.mean))
    cs_a, cs_b = engine.column_sum(D, 0, pl), g.column_sum([D], 0, pl)
    assert cs_a == cs_b
    g.close()


@pytest.mark.parametrize("mode", ["fused", "copy"])
@pytest.mark.parametrize("W", [2, 3, 5, 8])
def test_group_exchange_bit_identical(engine, tmp_path, W, mode, monkeypatch):
    """W members on one GPU: per-member shards, the exchange (fused: every member's K3a and scan
    write its slot of member 0's gather buffer directly; copy: member buffers copied into it), the
    device K3b over W rank buffers — the single-device bits (fast mode, reference order,
    Binary32Diagnostic), and the same for host / file sources every member streams its own
    ranges from."""
    from paper_2604_23826_b200 import Engine

    monkeypatch.setenv("SSTAT_GROUP_EXCHANGE", mode)
    n, p, chunk = 300_007, 16, 4099
    D = gen(engine, n, p)
    pl = plan(n, chunk)
    g = Engine(devices=[0] * W)
    parts = shards(D, pl, W)
    for flags, prec in ((0, 0), (2, 0), (0, 1)):
        pp = plan(n, chunk, prec)
        want = engine.dataset_suffstats(D, schema(p), pp, flags=flags)
        assert g.dataset_suffstats(parts, schema(p), pp, flags=flags).bit_equal(want), (flags, prec)
    want = engine.dataset_suffstats(D, schema(p), pl)
    H = D.cpu().numpy()
    assert g.dataset_suffstats(H, schema(p), pl).bit_equal(want)
    path = tmp_path / "g.bin"
    hdr = bytearray(64)
    hdr[0:8] = b"SSTATBIN"
    hdr[8:12] = (1).to_bytes(4, "little")
    hdr[12:20] = n.to_bytes(8, "little")
    hdr[20:24] = p.to_bytes(4, "little")
    with open(path, "wb") as f:
        f.write(hdr)
        H.tofile(f)
    assert g.dataset_suffstats(str(path), schema(p), pl).bit_equal(want)
    # the passes next to the path
    cm_a, cm_b = engine.comoments(D, schema(p), pl), g.comoments(parts, schema(p), pl)
    assert np.array_equal(bits(cm_a.m2), bits(cm_b.m2)) and np.array_equal(bits(cm_a.mean), bits(cm_b.mean))
    for flags in (0, 2):
        assert engine.column_sum(D, 1, pl, flags=flags) == g.column_sum(parts, 1, pl, flags=flags)
    g.close()


@pytest.mark.parametrize("p", [72, 256])
def test_group_wide_p_bit_identical(engine, p):
    """K1w / K2 widths through a 3-member group."""
    from paper_2604_23826_b200 import Engine

    n, chunk = 120_001, 33_333
    D = gen(engine, n, p, kind=2, seed=9)
    pl = plan(n, chunk)
    want = engine.dataset_suffstats(D, schema(p), pl)
    g = Engine(devices=[0, 0, 0])
    assert g.dataset_suffstats(shards(D, pl, 3), schema(p), pl).bit_equal(want)
    g.close()


@pytest.mark.parametrize("mode", ["fused", "copy"])
def test_group_nonfinite_reports_lowest_range(engine, mode, monkeypatch):
    """Non-finite values on two members: every member scans before the exchange, the rank
    headers meet in member 0, and the error is the single-device one (lowest failing range,
    its first non-finite row / column, reduce.hpp:111-134)."""
    from paper_2604_23826_b200 import Engine, ReductionError

    monkeypatch.setenv("SSTAT_GROUP_EXCHANGE", mode)

    torch = torch_mod()
    n, p, chunk = 100_000, 16, 1000
    D = gen(engine, n, p)
    D[77_777, 3] = float("nan")
    D[41_001, 9] = float("inf")
    pl = plan(n, chunk)
    with pytest.raises(ReductionError) as want:
        engine.dataset_suffstats(D, schema(p), pl)
    g = Engine(devices=[0] * 4)
    with pytest.raises(ReductionError) as got:
        g.dataset_suffstats(shards(D, pl, 4), schema(p), pl)
    assert got.value.range_index() == want.value.range_index() == 41
    assert str(got.value) == str(want.value)
    assert got.value.cause.row() == 41_001 and got.value.cause.column() == 9
    # the group recovers: a clean call after the failure
    D[77_777, 3] = 0.0
    D[41_001, 9] = 0.0
    torch.cuda.synchronize()
    assert g.dataset_suffstats(shards(D, pl, 4), schema(p), pl).bit_equal(engine.dataset_suffstats(D, schema(p), pl))
    g.close()


@pytest.mark.parametrize("mode", ["fused", "copy"])
def test_group_member_failure_is_published(engine, mode, monkeypatch):
    """A member whose local phase fails (its shard does not cover its ranges) publishes its
    status in its rank header; the exchange and fold still run, the rank headers name that
    member (the group checks them against the host-side failures), and the call raises the
    member's own error — the path a failing rank of a multi-process run takes instead of
    leaving its peers in the collective.  The next call succeeds."""
    from paper_2604_23826_b200 import Engine

    monkeypatch.setenv("SSTAT_GROUP_EXCHANGE", mode)

    n, p, chunk = 90_000, 16, 3000
    D = gen(engine, n, p)
    pl = plan(n, chunk)
    g = Engine(devices=[0, 0, 0])
    parts = shards(D, pl, 3)
    short = [parts[0], parts[1][:-5].contiguous(), parts[2]]
    with pytest.raises(ValueError, match="do not cover"):
        g.dataset_suffstats(short, schema(p), pl)
    with pytest.raises(ValueError, match="do not cover"):
        g.column_sum(short, 0, pl)
    with pytest.raises(ValueError, match="do not cover"):
        g.comoments(short, schema(p), pl)
    assert g.dataset_suffstats(parts, schema(p), pl).bit_equal(engine.dataset_suffstats(D, schema(p), pl))
    g.close()


def test_stream_ordering_without_sync():
    """A CUDA tensor written by an asynchronous torch kernel and passed straight in (no
    synchronize): the engine follows torch's current stream, so it reads the finished data
    (the context stream was not ordered after the producer)."""
    from paper_2604_23826_b200 import Engine

    torch = torch_mod()
    n, p = 4_000_000, 16
    e = Engine(0)
    X = torch.empty((n, p), dtype=torch.float64, device="cuda")
    e.generate(X, 0, 5, 1.0, 2, 0, n, p)
    want = e.dataset_suffstats(X, schema(p), plan(n, 1 << 20))
    e.close()
    for use_side_stream in (False, True):
        e = Engine(0)
        s = torch.cuda.Stream() if use_side_stream else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            D = torch.zeros((n, p), dtype=torch.float64, device="cuda")
            for _ in range(3):  # keep the producer busy long after the call is enqueued
                D.copy_(X)
                D.mul_(1.0)
            got = e.dataset_suffstats(D, schema(p), plan(n, 1 << 20))
        assert got.bit_equal(want), use_side_stream
        e.close()


@pytest.mark.parametrize("p", [40, 129])
def test_reference_order_streams_ranges_in_pieces(engine, tmp_path, oracle, p):
    """Reference-order mode from host / file sources with ranges larger than a staging slot:
    each range streams in pieces whose chains continue across launches — bit-identical to the
    device-resident pass and to the reference's sequential order (such ranges used
    to fail with 'staging slot smaller than one work unit').  column_sum's sequential mode too."""
    from paper_2604_23826_b200 import Engine

    n, chunk = 70_001 if p == 40 else 20_001, 1 << 15
    D = gen(engine, n, p, kind=2, seed=4)
    pl = plan(n, chunk)
    want = engine.dataset_suffstats(D, schema(p), pl, flags=2)
    H = D.cpu().numpy()
    e = Engine(0)
    e.set_staging(2, 1 << 20)  # a 2^15-row range at p = 40 is 10 MiB: 10+ pieces
    assert e.dataset_suffstats(H, schema(p), pl, flags=2).bit_equal(want)
    pl32 = plan(n, chunk, 1)
    assert e.dataset_suffstats(H, schema(p), pl32).bit_equal(engine.dataset_suffstats(D, schema(p), pl32))
    s, c = oracle.plan_partitions(n, chunk)
    _, ws, wS = oracle.run_reduction(H, p, s, c, 4)
    assert np.array_equal(bits(want.cross), bits(wS)) and np.array_equal(bits(want.sums), bits(ws))
    for prec in (0, 1):
        a = engine.column_sum(D, 3, plan(n, chunk, prec), flags=2)
        b = e.column_sum(H, 3, plan(n, chunk, prec), flags=2)
        assert a == b, prec
    e.close()


def test_wide_fast_path_tiles_larger_than_a_slot(engine):
    """p = 1100 from host memory: one K2 tile (32768 rows) is 288 MB, over the default 256 MiB
    slot; the ring grows its slots to the tile instead of failing."""
    n, p = 40_000, 1100
    D = gen(engine, n, p, kind=2, seed=8)
    pl = plan(n, 1 << 20)
    want = engine.dataset_suffstats(D, schema(p), pl)
    got = engine.dataset_suffstats(D.cpu().numpy(), schema(p), pl)
    assert got.bit_equal(want)


def test_reader_source(engine):
    """SSTAT_SRC_READER (BinaryReader::read_rows as a callback): rows served by filling the
    pinned scratch slot, or by pointing at pinned memory the caller owns, give the bits of the
    host-array source; a failing callback surfaces as IoError."""
    from paper_2604_23826_b200 import Engine, IoError, RowReader

    n, p, chunk = 600_001, 16, 1 << 17
    D = gen(engine, n, p)
    pl = plan(n, chunk)
    want = engine.dataset_suffstats(D, schema(p), pl)
    H = D.cpu().pin_memory()
    A = H.numpy()
    calls = []

    def fill(row, k, scratch):
        calls.append((row, k))
        ctypes.memmove(scratch, A[row:row + k].ctypes.data, k * p * 8)
        return scratch

    def point(row, k, scratch):
        return H.data_ptr() + row * p * 8

    e = Engine(0)
    e.set_staging(3, 4 << 20)
    for fn in (fill, point):
        for flags in (0, 2):
            got = e.dataset_suffstats(RowReader(fn, n), schema(p), pl, flags=flags)
            assert got.bit_equal(engine.dataset_suffstats(D, schema(p), pl, flags=flags)), (fn.__name__, flags)
    assert calls and all(k * p * 8 <= 4 << 20 for _, k in calls)

    def broken(row, k, scratch):
        if row > n // 2:
            raise OSError("disk gone")
        return fill(row, k, scratch)

    with pytest.raises(IoError, match="disk gone"):
        e.dataset_suffstats(RowReader(broken, n), schema(p), pl)
    assert e.dataset_suffstats(RowReader(point, n), schema(p), pl).bit_equal(want)
    e.close()


@pytest.mark.parametrize("n,chunk", [(1_000_000, 1 << 20), (300_000, 100_000), (5_000, 1 << 20)])
def test_small_plans_match_the_reference(engine, oracle, n, chunk):
    """Plans too small for 4096-row tiles (C1's shape and smaller): K1 cuts shorter tiles and reads
    each range's shift row in place, K3a folds long ranges over a cluster, a one-range plan skips
    K3b — the fast path stays within tolerance of the reference order and bit-exact on the integer
    columns; an all -0.0 column gives +0.0 sums like the reference's fold from +0.0; a non-finite
    value reports the single-range error."""
    from paper_2604_23826_b200 import ReductionError

    torch = torch_mod()
    p = 9
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 1, 42, 1.0, 0, 0, n, p)  # column 0 = row number (integer)
    D[:, 5] = -0.0
    pl = plan(n, chunk)
    fast = engine.dataset_suffstats(D, schema(p), pl)
    X = D.cpu().numpy()
    s, c = oracle.plan_partitions(n, chunk)
    _, ws, wS = oracle.run_reduction(X, p, s, c, 8)
    assert np.array_equal(bits(fast.sums[[0, 5]]), bits(ws[[0, 5]]))
    assert bits(fast.sums[5:6])[0] == 0  # +0.0
    assert cs_err(fast.cross, wS, p) <= 1e-12 or n * (n + 1) * (2 * n + 1) // 6 > 2**53
    exact = engine.dataset_suffstats(D, schema(p), pl, flags=2)
    assert np.array_equal(bits(exact.cross), bits(wS)) and np.array_equal(bits(exact.sums), bits(ws))
    D[n // 3, 7] = float("nan")
    with pytest.raises(ReductionError) as e:
        engine.dataset_suffstats(D, schema(p), pl)
    assert e.value.cause.row() == n // 3 and e.value.cause.column() == 7
    assert e.value.range_index() == (n // 3) // chunk


def test_group_member0_state_after_fused_calls(engine):
    """The fused exchange leaves member 0's own rank buffer alone: a chunk with a non-finite value
    accumulated through the group, then a fused dataset pass, then a clean chunk — each call
    reports exactly its own outcome (no stale error header)."""
    import torch

    from paper_2604_23826_b200 import Chunk, Engine, NonFiniteError

    g = Engine(devices=[0, 0])
    p = 8
    bad = torch.ones((100, p), dtype=torch.float64, device="cuda")
    bad[40, 3] = float("inf")
    with pytest.raises(NonFiniteError):
        g.accumulate_chunk(Chunk(0, 100, p, bad), schema(p))
    n = 50_000
    D = gen(engine, n, p, kind=2)
    pl = plan(n, 5_000)
    assert g.dataset_suffstats(shards(D, pl, 2), schema(p), pl).bit_equal(engine.dataset_suffstats(D, schema(p), pl))
    good = torch.ones((100, p), dtype=torch.float64, device="cuda")
    assert g.accumulate_chunk(Chunk(0, 100, p, good), schema(p)).n == 100
    g.close()


def test_group_reader_and_pieces(engine, tmp_path):
    """A device group reading a RowReader (both members call it, each for its own ranges) and a
    file in reference order through slots smaller than a range (pieces per member): the
    single-device bits."""
    from paper_2604_23826_b200 import Engine, RowReader

    n, p, chunk = 200_003, 40, 1 << 15
    D = gen(engine, n, p, kind=2, seed=12)
    pl = plan(n, chunk)
    H = D.cpu().numpy()
    calls = []

    def read(row, k, scratch):
        calls.append(row)
        ctypes.memmove(scratch, H[row:row + k].ctypes.data, k * p * 8)
        return scratch

    path = tmp_path / "gp.bin"
    hdr = bytearray(64)
    hdr[0:8] = b"SSTATBIN"
    hdr[8:12] = (1).to_bytes(4, "little")
    hdr[12:20] = n.to_bytes(8, "little")
    hdr[20:24] = p.to_bytes(4, "little")
    with open(path, "wb") as f:
        f.write(hdr)
        H.tofile(f)
    g = Engine(devices=[0, 0, 0])
    g.set_staging(2, 1 << 20)
    for flags in (0, 2):
        want = engine.dataset_suffstats(D, schema(p), pl, flags=flags)
        assert g.dataset_suffstats(RowReader(read, n), schema(p), pl, flags=flags).bit_equal(want), flags
        assert g.dataset_suffstats(str(path), schema(p), pl, flags=flags).bit_equal(want), flags
    assert min(calls) == 0 and max(calls) > n // 2  # every member read its own ranges
    g.close()


def test_group_and_explicit_stream_ordering_without_sync(engine):
    """Shards written by asynchronous torch kernels on a side stream reach a device group (whose
    members launch on their own streams) only after the producer is done; an engine bound with
    set_stream to the producer's stream is ordered after it on the device."""
    from paper_2604_23826_b200 import Engine

    torch = torch_mod()
    n, p = 4_000_000, 16
    pl = plan(n, 1 << 20)
    X = gen(engine, n, p, seed=9)
    torch.cuda.synchronize()
    want = engine.dataset_suffstats(X, schema(p), pl)
    s = torch.cuda.Stream()
    g = Engine(devices=[0, 0])
    e = Engine(0)
    e.set_stream(s.cuda_stream)
    assert g.n_devices == 2 and e.n_devices == 1
    try:
        with torch.cuda.stream(s):
            D = torch.zeros((n, p), dtype=torch.float64, device="cuda")
            for _ in range(3):
                D.copy_(X)
                D.mul_(1.0)
            parts = shards(D, pl, 2)
            got_g = g.dataset_suffstats(parts, schema(p), pl)
        assert got_g.bit_equal(want)
        with torch.cuda.stream(s):
            for _ in range(3):
                D.mul_(1.0)
            got_e = e.dataset_suffstats(D, schema(p), pl)
        assert got_e.bit_equal(want)
    finally:
        g.close()
        e.close()
