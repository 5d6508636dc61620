"""Timings are filled only when the caller asks for them, like the reference's optional
ReductionTimings* (reduce.hpp:70-73): an untimed call replays a graph without event nodes and
leaves last_timings empty; a timed one reports the accumulate kernel, its launches and bytes.
The result bits do not depend on whether the call was timed."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rows(engine, n, p, kind=0, n_int=2, seed=11):
    import torch

    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, kind, seed, 1.0, n_int, 0, n, p)
    torch.cuda.synchronize()
    return D


@pytest.mark.parametrize("n,p,chunk,launches", [(200_000, 9, 1 << 20, 2),   # small plan, one range: K1 K3a
                                                (1_500_000, 16, 1 << 20, 3),  # small plan: K1 K3a K3b
                                                (6_000_000, 16, 1 << 20, 4)])  # full tiles: gather K1 K3a K3b
def test_timings_only_when_asked(engine, n, p, chunk, launches):
    from paper_2604_23826_b200 import DatasetSchema, ReductionPlan, ReductionTimings, plan_partitions

    D = rows(engine, n, p)
    plan = ReductionPlan(plan_partitions(n, chunk))
    sc = DatasetSchema.generic(p, False)
    assert engine.collect_timings is False
    a = engine.dataset_suffstats(D, sc, plan)
    assert engine.last_timings is None
    t = ReductionTimings()
    b = engine.dataset_suffstats(D, sc, plan, timings=t)
    assert t.bytes_read == n * p * 8 and t.work_seconds > 0 and t.kernel_launches == launches
    assert engine.last_timings.kernel.decode().startswith("k_smallp")
    c = engine.dataset_suffstats(D, sc, plan)
    assert engine.last_timings is None
    assert a.bit_equal(b) and a.bit_equal(c)
    engine.collect_timings = True
    try:
        d = engine.dataset_suffstats(D, sc, plan)
        assert engine.last_timings.kernel_seconds > 0 and d.bit_equal(a)
    finally:
        engine.collect_timings = False


def test_host_source_timings(engine):
    """A pinned host source reports its H2D time and bytes; untimed, the same bits."""
    import torch

    from paper_2604_23826_b200 import DatasetSchema, ReductionPlan, ReductionTimings, plan_partitions

    n, p = 2_000_000, 16
    D = rows(engine, n, p)
    H = torch.empty((n, p), dtype=torch.float64, pin_memory=True)
    H.copy_(D)
    plan = ReductionPlan(plan_partitions(n, 1 << 18))
    sc = DatasetSchema.generic(p, False)
    t = ReductionTimings()
    a = engine.dataset_suffstats(H, sc, plan, timings=t)
    assert t.read_seconds > 0 and t.bytes_read == n * p * 8
    b = engine.dataset_suffstats(H, sc, plan)
    assert a.bit_equal(b) and a.bit_equal(engine.dataset_suffstats(D, sc, plan))
    assert np.isfinite(a.cross).all()
    # a device group of two members, each streaming its ranges of the same pinned array: the
    # longest member copy span
    from paper_2604_23826_b200 import Engine

    g = Engine(devices=[0, 0])
    try:
        tg = ReductionTimings()
        assert g.dataset_suffstats(H, sc, plan, timings=tg).bit_equal(a)
        assert tg.read_seconds > 0 and tg.bytes_read == n * p * 8
    finally:
        g.close()
