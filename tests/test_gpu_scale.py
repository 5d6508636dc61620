"""Parity at BASELINE scale against the reference itself (oracle/_ref: the unmodified reference
library compiled from /root/reference/proj/src, shipped prebuilt to the GPU box), not against
the GPU's own reference-order mode.

  * C2 in full: the 1e8 x 16 SSTATBIN bytes (12.8 GB in /dev/shm), the reference's
    dataset_suffstats on all host threads (plan_partitions(n, 2^20): 96 ranges) against the
    GPU fast path and reference-order mode on the same bytes, and the reference's own
    analyze / run_pca on both results (reference src/suffstats.cpp:279-288, analysis.cpp,
    pca.cpp).
  * C5's width: p = 256 over 2.5e6 rows at chunk 2^18 — 10 ranges of 8 K2 tiles (32768 rows)
    each, so the multi-tile, multi-range K2 path with its idle-slot side launch is checked
    against the reference, not only the 3000-row golden case.

Bars (BASELINE.json north_star): counts exact; integer-valued columns
bit-exact; sums / X^T X / covariance Cauchy-Schwarz-normalised <= 1e-12; correlation 1e-12
absolute; eigenvalues 1e-10 relative; reference-order mode bit-identical.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import bits, cs_err, sums_err

pytestmark = pytest.mark.gpu

TOL = 1e-12


def shm_path(name):
    d = "/dev/shm" if os.path.isdir("/dev/shm") else "/tmp"
    return os.path.join(d, f"{name}_{os.getpid()}.bin")


def write_sstatbin(path, H):
    n, p = H.shape
    hdr = bytearray(64)
    hdr[0:8] = b"SSTATBIN"
    hdr[8:12] = (1).to_bytes(4, "little")
    hdr[12:20] = int(n).to_bytes(8, "little")
    hdr[20:24] = int(p).to_bytes(4, "little")
    with open(path, "wb") as f:
        f.write(hdr)
        H.tofile(f)


def downstream_close(reference, p, ids, got, want_n, want_sums, want_cross):
    """The reference's analyze (mean / cov / corr) and run_pca on both results."""
    m_a, cov_a, corr_a = reference.analyze(p, ids, got.n, got.sums, got.cross)
    m_b, cov_b, corr_b = reference.analyze(p, ids, want_n, want_sums, want_cross)
    scale = np.sqrt(np.outer(np.diag(cov_b), np.diag(cov_b)))
    assert np.max(np.abs(cov_a - cov_b) / scale) <= TOL
    assert np.max(np.abs(corr_a - corr_b)) <= TOL
    for basis in (0, 1):
        ev_a = reference.run_pca(p, ids, got.n, got.sums, got.cross, basis=basis)
        ev_b = reference.run_pca(p, ids, want_n, want_sums, want_cross, basis=basis)
        assert np.max(np.abs(ev_a - ev_b) / np.abs(ev_b)) <= 1e-10


def test_c2_full_size_vs_reference(engine, reference):
    import torch

    from paper_2604_23826_b200 import DatasetSchema, ReductionPlan, plan_partitions

    n, p = 100_000_000, 16
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 0, 42, 1.0, 2, 0, n, p)
    pl = ReductionPlan(plan_partitions(n, 1 << 20))
    sc = DatasetSchema.generic(p, False)
    fast = engine.dataset_suffstats(D, sc, pl)
    exact = engine.dataset_suffstats(D, sc, pl, flags=2)
    H = D.cpu().numpy()
    del D
    torch.cuda.empty_cache()
    path = shm_path("c2_parity")
    try:
        write_sstatbin(path, H)
        del H
        wn, ws, wS = reference.dataset_suffstats(path, p, 1 << 20, os.cpu_count() or 1)
        # the reference's call shape through the GPU: the same bits as the resident pass
        assert engine.dataset_suffstats(path, sc, pl).bit_equal(fast)
    finally:
        os.remove(path)
    assert fast.n == exact.n == wn == n
    # reference-order mode: bit-identical to the reference on all 152 entries
    assert np.array_equal(bits(exact.sums), bits(ws)) and np.array_equal(bits(exact.cross), bits(wS))
    # fast path: integer block (columns 0-1, rand_between(1, 100)) bit-exact, the rest in tolerance
    assert np.array_equal(bits(fast.sums[:2]), bits(ws[:2]))
    idx = [0, 1, p]  # (0,0), (0,1), (1,1)
    assert np.array_equal(bits(fast.cross[idx]), bits(wS[idx]))
    assert cs_err(fast.cross, wS, p) <= TOL
    assert sums_err(fast.sums, ws, wS, n, p) <= TOL
    downstream_close(reference, p, [], fast, wn, ws, wS)


def test_wide_p256_multi_range_multi_tile_vs_reference(engine, reference):
    import torch

    from paper_2604_23826_b200 import DatasetSchema, ReductionPlan, plan_partitions

    n, p, chunk = 2_500_000, 256, 1 << 18
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 2, 23, 1.0, 0, 0, n, p)
    pl = ReductionPlan(plan_partitions(n, chunk))
    assert len(pl.partition.ranges) == 10  # 9 x 2^18 rows (8 K2 tiles each) + a 140800-row tail
    sc = DatasetSchema.generic(p, False)
    engine.collect_timings = True
    try:
        fast = engine.dataset_suffstats(D, sc, pl)
    finally:
        engine.collect_timings = False
    kernel = engine.last_timings.kernel.decode()
    assert kernel.startswith("k_widep"), kernel
    H = D.cpu().numpy()
    del D
    torch.cuda.empty_cache()
    path = shm_path("p256_parity")
    try:
        write_sstatbin(path, H)
        del H
        wn, ws, wS = reference.dataset_suffstats(path, p, chunk, os.cpu_count() or 1)
        assert engine.dataset_suffstats(path, sc, pl).bit_equal(fast)  # file source, staged tiles
    finally:
        os.remove(path)
    assert fast.n == wn == n
    assert cs_err(fast.cross, wS, p) <= TOL
    assert sums_err(fast.sums, ws, wS, n, p) <= TOL
    downstream_close(reference, p, [], fast, wn, ws, wS)
