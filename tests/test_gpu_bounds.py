"""Memory-safety checks of our own (compute-sanitizer is closed on the GPU pool:
profiles/r02_sanitizer_closed.log).

  * Reads stay inside the rows they are given: every kernel family runs on a shard that sits
    between NaN guard rows in the same allocation (and at odd element offsets, so the unaligned
    staging paths run too).  A single read past either end would turn a sum into NaN and the call
    into a ReductionError; instead the result must be bit-identical to the same rows in a fresh
    allocation.
  * Writes stay inside the caller's output arrays: the raw C ABI writes into arrays surrounded by
    sentinel values, which must be intact afterwards.
"""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu


def schema(p):
    from paper_2604_23826_b200 import DatasetSchema

    return DatasetSchema.generic(p, False)


def plan(n, chunk, precision=0):
    from paper_2604_23826_b200 import PrecisionMode, ReductionPlan, plan_partitions

    return ReductionPlan(plan_partitions(n, chunk), 1, PrecisionMode(precision))


def guarded(engine, n, p, pad_rows, shift_elems, seed):
    """(clean, guarded): the same n x p rows in their own allocation and inside a NaN-filled
    one, starting shift_elems doubles past a row boundary of the guard region."""
    import torch

    clean = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(clean, 2, seed, 0.5, 0, 0, n, p)
    total = (2 * pad_rows + n) * p + 2 * shift_elems + 2
    buf = torch.full((total,), float("nan"), dtype=torch.float64, device="cuda")
    start = pad_rows * p + shift_elems
    view = buf[start:start + n * p].view(n, p)
    view.copy_(clean)
    torch.cuda.synchronize()
    return clean, view


@pytest.mark.parametrize("p", [1, 3, 9, 16, 17, 33, 64, 65, 72, 100, 128, 129, 256, 259])
@pytest.mark.parametrize("shift_elems", [0, 1])
def test_reads_stay_inside_the_shard(engine, p, shift_elems):
    n, chunk = 12_345 if p <= 128 else 70_001, 4_099 if p <= 128 else 33_333
    clean, view = guarded(engine, n, p, pad_rows=37, shift_elems=shift_elems, seed=p)
    pl = plan(n, chunk)
    for flags in (0, 2):
        want = engine.dataset_suffstats(clean, schema(p), pl, flags=flags)
        got = engine.dataset_suffstats(view, schema(p), pl, flags=flags)
        assert np.all(np.isfinite(got.cross)) and got.bit_equal(want), (p, shift_elems, flags)
    a, b = engine.comoments(clean, schema(p), pl), engine.comoments(view, schema(p), pl)
    assert np.array_equal(bits(a.m2), bits(b.m2))
    assert engine.column_sum(view, p - 1, pl) == engine.column_sum(clean, p - 1, pl)
    # one chunk (accumulate_chunk) over the same rows
    from paper_2604_23826_b200 import Chunk

    ca = engine.accumulate_chunk(Chunk(0, n, p, clean), schema(p))
    cb = engine.accumulate_chunk(Chunk(0, n, p, view), schema(p))
    assert ca.bit_equal(cb)


@pytest.mark.parametrize("p", [16, 72, 256])
def test_host_staging_reads_stay_inside_the_rows(engine, p):
    """The staged sources copy exactly the requested rows: a host array between NaN guard rows,
    passed as a view, streams through small slots with the same bits as the device pass."""
    from paper_2604_23826_b200 import Engine

    n, chunk = 50_001, 7_001
    clean, _ = guarded(engine, n, p, pad_rows=1, shift_elems=0, seed=7)
    host = np.full(((n + 40) * p + 1,), np.nan)
    view = host[20 * p + 1:20 * p + 1 + n * p].reshape(n, p)  # 8 bytes off 16-byte alignment
    view[:] = clean.cpu().numpy()
    e = Engine(0)
    e.set_staging(2, 1 << 20)
    for flags in (0, 2):
        want = engine.dataset_suffstats(clean, schema(p), plan(n, chunk), flags=flags)
        assert e.dataset_suffstats(view, schema(p), plan(n, chunk), flags=flags).bit_equal(want), flags
    e.close()


def test_outputs_written_inside_their_arrays(engine):
    """sstat_cuda_dataset / _accumulate / _comoments / _column_sum / _range_partials write exactly
    their outputs: sentinels on both sides of every output array survive the calls."""
    import torch

    from paper_2604_23826_b200 import _native as N

    lib = N.load()
    n, p = 30_000, 24
    E = p + p * (p + 1) // 2
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 2, 3, 1.0, 0, 0, n, p)
    starts = np.arange(0, n, 4096, dtype=np.uint64)
    counts = np.minimum(4096, n - starts).astype(np.uint64)
    R = len(starts)
    G = 64  # guard doubles per side
    SENT = -1.2345e300

    def guarded_out(k):
        a = np.full(k + 2 * G, SENT)
        return a, a[G:G + k]

    def intact(a, k):
        return np.all(a[:G] == SENT) and np.all(a[G + k:] == SENT)

    src = N.Source(kind=N.SRC_DEVICE, ptr=D.data_ptr(), first_row=0, n_rows=n)
    dp = ctypes.POINTER(ctypes.c_double)
    sa, s = guarded_out(p)
    ca, c = guarded_out(E - p)
    nn = ctypes.c_uint64()
    err = N.Error()
    tm = N.Timings()
    st = lib.sstat_cuda_dataset(engine._ctx, ctypes.byref(src), p, starts.ctypes.data, counts.ctypes.data, R, 0, 0,
                                ctypes.byref(nn), s.ctypes.data, c.ctypes.data, ctypes.byref(tm), ctypes.byref(err))
    assert st == 0 and intact(sa, p) and intact(ca, E - p) and np.all(np.isfinite(c))
    sa2, s2 = guarded_out(p)
    ca2, c2 = guarded_out(E - p)
    st = lib.sstat_cuda_accumulate(engine._ctx, ctypes.c_void_p(D.data_ptr()), n, p, 0, 0, 0, ctypes.byref(nn),
                                   s2.ctypes.data_as(dp), c2.ctypes.data_as(dp), ctypes.byref(err))
    assert st == 0 and intact(sa2, p) and intact(ca2, E - p)
    ma, m = guarded_out(p)
    m2a, m2 = guarded_out(E - p)
    st = lib.sstat_cuda_comoments(engine._ctx, ctypes.byref(src), p, starts.ctypes.data, counts.ctypes.data, R, 0,
                                  ctypes.byref(nn), m.ctypes.data_as(dp), m2.ctypes.data_as(dp), ctypes.byref(err))
    assert st == 0 and intact(ma, p) and intact(m2a, E - p)
    pa, part = guarded_out(3 * E)
    st = lib.sstat_cuda_range_partials(engine._ctx, ctypes.byref(src), p, starts.ctypes.data, counts.ctypes.data, R,
                                       2, 5, 0, 0, part.ctypes.data_as(dp), ctypes.byref(err))
    assert st == 0 and intact(pa, 3 * E) and np.all(np.isfinite(part))
    raw = (ctypes.c_char * (ctypes.sizeof(N.ColumnSum) + 2 * 64))()
    ctypes.memset(raw, 0x5A, len(raw))
    res = N.ColumnSum.from_buffer(raw, 64)
    st = lib.sstat_cuda_column_sum(engine._ctx, ctypes.byref(src), p, 3, starts.ctypes.data, counts.ctypes.data, R,
                                   0, 0, ctypes.byref(res), ctypes.byref(err))
    assert st == 0
    assert bytes(raw[:64]) == b"\x5a" * 64 and bytes(raw[64 + ctypes.sizeof(N.ColumnSum):]) == b"\x5a" * 64
