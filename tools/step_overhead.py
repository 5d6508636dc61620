"""Where does a dataset_suffstats step spend time beyond K1?  (C2, HBM-resident)"""
import ctypes
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions
from paper_2604_23826_b200 import _native as N

n, p = 100_000_000, 16
eng = Engine(0)
eng.collect_timings = True
D = torch.empty((n, p), dtype=torch.float64, device="cuda")
eng.generate(D, 0, 42, 1.0, 2, 0, n, p)
plan = ReductionPlan(plan_partitions(n, 1 << 20))
schema = DatasetSchema.generic(p, False)
for _ in range(3):
    eng.dataset_suffstats(D, schema, plan)
torch.cuda.synchronize()

K = 50
t0 = time.perf_counter()
for _ in range(K):
    eng.dataset_suffstats(D, schema, plan)
py = (time.perf_counter() - t0) / K
kern = eng.last_timings.kernel_seconds
fold = eng.last_timings.fold_seconds

# raw C call with prebuilt arguments
lib = N.load()
src = N.Source(kind=N.SRC_DEVICE, ptr=D.data_ptr(), first_row=0, n_rows=n)
starts, counts = plan.partition.arrays()
sums, cross = np.zeros(p), np.zeros(p * (p + 1) // 2)
nn = ctypes.c_uint64()
tm, err = N.Timings(), N.Error()
dp = ctypes.POINTER(ctypes.c_double)
args = (eng._ctx, ctypes.byref(src), p, starts.ctypes.data, counts.ctypes.data, len(starts), 0, 0, ctypes.byref(nn),
        sums.ctypes.data_as(dp), cross.ctypes.data_as(dp), ctypes.byref(tm), ctypes.byref(err))
t0 = time.perf_counter()
for _ in range(K):
    lib.sstat_cuda_dataset(*args)
raw = (time.perf_counter() - t0) / K
print(f"python API step {py*1e3:.3f} ms | raw C call {raw*1e3:.3f} ms | K1 {kern*1e3:.3f} ms | folds {fold*1e3:.3f} ms "
      f"| total_seconds {tm.total_seconds*1e3:.3f} ms | launches {tm.kernel_launches}")
