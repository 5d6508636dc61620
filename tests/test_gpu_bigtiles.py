"""Large plans take K1 tiles of kBigTileRows = 16384 rows (common.cuh): the tile is still the
deterministic unit, so the resident, host-streamed and device-group passes give the same bits;
against the kTileRows = 4096 cut of the same rows (SSTAT_K1_TILE_ROWS) the integer-valued
columns stay exact and the rest agree to rounding."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import cs_err

pytestmark = pytest.mark.gpu

BIG = 8 * 148 * 4 * 16384  # kBigTileMin tiles of kBigTileRows: the smallest plan that takes them


@pytest.mark.parametrize("p", [9, 16, 40])
def test_big_tiles_bit_identical_across_sources_and_groups(engine, p):
    import torch

    from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions, shard_ranges

    n = BIG + 12_345  # ragged last range and tile
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 0, 100 + p, 1.0, 2, 0, n, p)
    torch.cuda.synchronize()
    plan = ReductionPlan(plan_partitions(n, 1 << 20))
    sc = DatasetSchema.generic(p, False)
    engine.collect_timings = True
    try:
        a = engine.dataset_suffstats(D, sc, plan)
        kernel = engine.last_timings.kernel.decode()
    finally:
        engine.collect_timings = False
    assert kernel.startswith("k_smallp") and "16384" in kernel, kernel
    b = engine.dataset_suffstats(D, sc, plan)  # untimed graph
    assert a.bit_equal(b)
    g = Engine(devices=[0, 0])  # two members: each its contiguous shard of the ranges (views)
    try:
        parts = []
        R = len(plan.partition.ranges)
        for i in range(2):
            f, l = shard_ranges(R, i, 2)
            r0 = plan.partition.ranges[f].start_row
            r1 = plan.partition.ranges[l - 1].start_row + plan.partition.ranges[l - 1].row_count
            parts.append(D[r0:r1])
        assert g.dataset_suffstats(parts, sc, plan).bit_equal(a)
    finally:
        g.close()
    # the 4096-row cut of the same rows
    os.environ["SSTAT_K1_TILE_ROWS"] = "4096"
    try:
        c = engine.dataset_suffstats(D, sc, plan)
    finally:
        del os.environ["SSTAT_K1_TILE_ROWS"]
    assert c.n == a.n == n
    assert np.array_equal(a.sums[:2], c.sums[:2])  # integer-valued columns: exact either way
    assert cs_err(a.cross, c.cross, p) < 1e-13
    assert np.max(np.abs(a.sums - c.sums) / np.maximum(np.abs(c.sums), 1.0)) < 1e-12
    if p == 16:  # the co-moments ride on the same K1 tiles: big against 4096-row
        m_big = engine.comoments(D, sc, plan)
        os.environ["SSTAT_K1_TILE_ROWS"] = "4096"
        try:
            m_4k = engine.comoments(D, sc, plan)
        finally:
            del os.environ["SSTAT_K1_TILE_ROWS"]
        assert m_big.n == m_4k.n == n
        assert np.max(np.abs(m_big.mean - m_4k.mean) / np.maximum(np.abs(m_4k.mean), 1.0)) < 1e-13
        assert cs_err(m_big.m2, m_4k.m2, p) < 1e-12
    # host-streamed (pinned, 4-slot ring): the same tiles, the same bits
    H = torch.empty((n, p), dtype=torch.float64, pin_memory=True)
    H.copy_(D)
    del D
    torch.cuda.empty_cache()
    assert engine.dataset_suffstats(H, sc, plan).bit_equal(a)


def test_plans_below_the_threshold_keep_4096_row_tiles(engine):
    import torch

    from paper_2604_23826_b200 import DatasetSchema, ReductionPlan, plan_partitions

    for n, p in [(BIG - 16384, 16), (BIG + 12_345, 8)]:  # one tile short; p <= 8
        D = torch.empty((n, p), dtype=torch.float64, device="cuda")
        engine.generate(D, 0, 7, 1.0, 2, 0, n, p)
        torch.cuda.synchronize()
        engine.collect_timings = True
        try:
            engine.dataset_suffstats(D, DatasetSchema.generic(p, False), ReductionPlan(plan_partitions(n, 1 << 20)))
            kernel = engine.last_timings.kernel.decode()
        finally:
            engine.collect_timings = False
        assert "4096" in kernel, (n, p, kernel)
        del D
        torch.cuda.empty_cache()
