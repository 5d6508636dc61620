"""C1 call time (device events and host clock over 2000 back-to-back calls) for one package tree:
    python tools/ab/c1_call.py <tree>"""
import os, sys, time
sys.path.insert(0, os.path.abspath(sys.argv[1]))
import torch
from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions
n, p = 1_000_000, 9
eng = Engine(0)
D = torch.empty((n, p), dtype=torch.float64, device="cuda")
eng.generate(D, 1, 42, 1.0, 0, 0, n, p)
plan = ReductionPlan(plan_partitions(n, 1 << 20))
sc = DatasetSchema.generic(p, True)
s = torch.cuda.current_stream()
for rep in range(3):
    for _ in range(50): eng.dataset_suffstats(D, sc, plan)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record(s)
    for _ in range(2000): eng.dataset_suffstats(D, sc, plan)
    b.record(s); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(sys.argv[1], os.environ.get("SSTAT_EXP_NOCOPY", "-"), f"device {a.elapsed_time(b)/2000*1e3:.1f} us host {(t1-t0)/2000*1e6:.1f} us")
