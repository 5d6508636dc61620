"""Run dataset_suffstats on one HBM-resident synthetic case (for ncu captures).
    python tools/one_case.py p rows [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions  # noqa: E402

p, n = int(sys.argv[1]), int(float(sys.argv[2]))
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
eng = Engine(0)
eng.collect_timings = True
D = torch.empty((n, p), dtype=torch.float64, device="cuda")
eng.generate(D, 2, 1, 1.0, 0, 0, n, p)
plan = ReductionPlan(plan_partitions(n, 1 << 20))
for _ in range(steps):
    eng.dataset_suffstats(D, DatasetSchema.generic(p, False), plan)
    print(p, n, eng.last_timings.kernel_seconds * 1e3, "ms", flush=True)
