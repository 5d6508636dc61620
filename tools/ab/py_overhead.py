"""Python-side cost per piece of a small dataset_suffstats call (C1): python tools/ab/py_overhead.py"""
import sys, time, timeit
sys.path.insert(0, '/root/repo')
import torch
from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions
n, p = 1_000_000, 9
eng = Engine(0)
D = torch.empty((n, p), dtype=torch.float64, device="cuda")
eng.generate(D, 1, 42, 1.0, 0, 0, n, p)
plan = ReductionPlan(plan_partitions(n, 1 << 20))
sc = DatasetSchema.generic(p, True)
eng.dataset_suffstats(D, sc, plan)
K = 20000
def t(f, k=K):
    f()
    t0 = time.perf_counter()
    for _ in range(k): f()
    return (time.perf_counter() - t0) / k * 1e6
print("current_stream().cuda_stream", t(lambda: torch.cuda.current_stream(D.device).cuda_stream))
print("_cuda_getCurrentRawStream", t(lambda: torch._C._cuda_getCurrentRawStream(0)))
print("D.device.index", t(lambda: D.device.index))
print("schema.validate", t(lambda: sc.validate()))
print("_source", t(lambda: eng._source(D, p, 0, None, plan)))
print("addresses", t(lambda: plan.partition.addresses()))
print("data_ptr", t(lambda: D.data_ptr()))
print("is_contiguous", t(lambda: D.is_contiguous()))
print("full call", t(lambda: eng.dataset_suffstats(D, sc, plan), 3000))
