"""Multi-rank host logic on CPU (torch.distributed gloo, world_size 2 and 3).

The GPU path shards the plan's ranges contiguously over ranks (sstat_shard_ranges), each
rank writes [4-double header | its range partials] into a fixed-stride buffer, the
buffers are all-gathered (NCCL on the GPU box) and every rank folds all ranges in
ascending order with the same fold code (fold_entry; sstat_fold_ranges_host on the
host).  Here the per-range partials come from the CPU oracle and the all-gather from
gloo, so the sharding, the layout, the error header and the fold are exercised exactly
as on the GPU, and the result must equal the single-process reference fold bit for bit.
"""
from __future__ import annotations

import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, bits


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_2604_23826_b200 import _native as N
        from paper_2604_23826_b200 import shard_ranges

        o = Oracle()
        n, p, chunk, poison = case
        X = o.generate(0, 11, 1.0, 2, 0, n, p)
        if poison is not None:
            X[poison[0], poison[1]] = np.nan
        starts, counts = o.plan_partitions(n, chunk)
        R, E = len(starts), p + p * (p + 1) // 2
        f, l = shard_ranges(R, rank, world)
        lmax = (R + world - 1) // world
        stride = 4 + lmax * E
        mine = np.zeros(stride)
        hdr = mine[:4].view(np.uint64)
        hdr[:] = np.iinfo(np.uint64).max
        for i in range(f, l):  # this rank's ranges: the per-range partials K3a produces
            r0, rc = int(starts[i]), int(counts[i])
            res = o.accumulate_chunk(X[r0:r0 + rc], p, r0)
            if res[0] == "nonfinite":
                if hdr[0] == np.iinfo(np.uint64).max:
                    hdr[0] = i
                    hdr[1] = res[1] * p + res[2]
                continue
            mine[4 + (i - f) * E: 4 + (i - f + 1) * E] = np.concatenate([res[1], res[2]])
        gathered = [torch.zeros(stride, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(mine))
        buf = torch.cat(gathered).numpy().copy()
        # error header: lowest failing range over ranks (ranges ascend with rank)
        lin = min(int(buf[q * stride + 1: q * stride + 2].view(np.uint64)[0]) for q in range(world))
        if lin != np.iinfo(np.uint64).max:
            row, col = lin // p, lin % p
            rng = int(np.searchsorted(starts, row, side="right") - 1)
            q.put((rank, "error", (rng, row, col)))
            return
        out = np.zeros(E)
        lib = N.load()
        dp = ctypes.POINTER(ctypes.c_double)
        assert lib.sstat_fold_ranges_host(buf.ctypes.data_as(dp), stride, R, world, p, 0, 2, out.ctypes.data_as(dp)) == 0
        q.put((rank, "ok", out))
    finally:
        dist.destroy_process_group()


def _run(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    return sorted(results, key=lambda r: r[0])


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fold_bit_identical_to_single_process(oracle, world):
    n, p, chunk = 40007, 7, 1931
    results = _run(world, (n, p, chunk, None))
    X = oracle.generate(0, 11, 1.0, 2, 0, n, p)
    s, c = oracle.plan_partitions(n, chunk)
    want = oracle.run_reduction(X, p, s, c, 3)
    for rank, kind, out in results:
        assert kind == "ok"
        assert np.array_equal(bits(out[:p]), bits(want[1])), rank
        assert np.array_equal(bits(out[p:]), bits(want[2])), rank


def test_sharded_error_reports_lowest_range_on_every_rank(oracle):
    n, p, chunk = 30000, 5, 1000
    results = _run(2, (n, p, chunk, (25000, 3)))
    X = oracle.generate(0, 11, 1.0, 2, 0, n, p)
    X[25000, 3] = np.nan
    s, c = oracle.plan_partitions(n, chunk)
    want = oracle.run_reduction(X, p, s, c, 2)
    assert want[0] == "nonfinite"
    for rank, kind, err in results:
        assert kind == "error"
        assert err == (want[1], want[2], want[3]) == (25, 25000, 3)
