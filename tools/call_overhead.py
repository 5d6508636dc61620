"""Host cost of one small synchronous pass (C1: 1e6 x 9, one range): the Python API call, the raw
C ABI call with prepared arguments, and the device time of the replayed graph, per call.
    python tools/call_overhead.py [K]"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions  # noqa: E402
from paper_2604_23826_b200 import _native as N  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
n, p = 1_000_000, 9
eng = Engine(0)
D = torch.empty((n, p), dtype=torch.float64, device="cuda")
eng.generate(D, 1, 42, 1.0, 0, 0, n, p)
plan = ReductionPlan(plan_partitions(n, 1 << 20))
sc = DatasetSchema.generic(p, True)
lib = N.load()
for timed in (False, True):
    eng.collect_timings = timed
    for _ in range(20):
        eng.dataset_suffstats(D, sc, plan)
    t0 = time.perf_counter()
    for _ in range(K):
        eng.dataset_suffstats(D, sc, plan)
    py = (time.perf_counter() - t0) / K
    # the raw ABI call with everything prepared once
    src = N.Source(kind=N.SRC_DEVICE, ptr=D.data_ptr(), first_row=0, n_rows=n)
    starts, counts = plan.partition.arrays()
    E = p + p * (p + 1) // 2
    out = np.zeros(E)
    nn, err, tm = ctypes.c_uint64(), N.Error(), N.Timings()
    args = (eng._ctx, ctypes.byref(src), p, starts.ctypes.data, counts.ctypes.data, len(starts), 0, 0, ctypes.byref(nn),
            out.ctypes.data, out.ctypes.data + 8 * p, ctypes.byref(tm) if timed else None, ctypes.byref(err))
    for _ in range(20):
        lib.sstat_cuda_dataset(*args)
    t0 = time.perf_counter()
    for _ in range(K):
        lib.sstat_cuda_dataset(*args)
    raw = (time.perf_counter() - t0) / K
    extra = f", device K1 {tm.kernel_seconds * 1e6:.1f} us + folds {tm.fold_seconds * 1e6:.1f} us" if timed else ""
    print(f"timings={'on ' if timed else 'off'}: Engine.dataset_suffstats {py * 1e6:.1f} us/call, raw C ABI call "
          f"{raw * 1e6:.1f} us/call{extra}", flush=True)
