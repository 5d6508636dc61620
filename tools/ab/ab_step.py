"""A/B of the C2 / C1 step between package trees: python tools/ab/ab_step.py <tree> [K]"""
import os, sys
tree = sys.argv[1]
sys.path.insert(0, os.path.abspath(tree))
import torch
from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions
K = int(sys.argv[2]) if len(sys.argv) > 2 else 100
for name, n, p, kind, n_int in (("C2", 100_000_000, 16, 0, 2), ("C1", 1_000_000, 9, 1, 0)):
    eng = Engine(0)
    eng.collect_timings = True
    s = torch.cuda.current_stream()
    eng.set_stream(s.cuda_stream)
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    eng.generate(D, kind, 42, 1.0, n_int, 0, n, p)
    plan = ReductionPlan(plan_partitions(n, 1 << 20))
    sc = DatasetSchema.generic(p, kind == 1)
    for rep in range(3):
        for _ in range(5):
            eng.dataset_suffstats(D, sc, plan)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(K):
            eng.dataset_suffstats(D, sc, plan)
        b.record(s)
        torch.cuda.synchronize()
        t = eng.last_timings
        print(f"{tree} {name} rep{rep} step {a.elapsed_time(b) / K * 1e3:.1f} us K1 {t.kernel_seconds * 1e6:.1f} us folds {t.fold_seconds * 1e6:.1f}", flush=True)
    del D
    eng.close()
    torch.cuda.empty_cache()
