"""Reference-order mode (SSTAT_FLAG_REFEXACT) throughput vs the fast mode, HBM-resident."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions  # noqa: E402

eng = Engine(0)
for n, p, chunk in ((100_000_000, 16, 1 << 20), (100_000_000, 16, 1 << 16), (1_000_000, 9, 1 << 20), (2_000_000, 256, 1 << 18)):
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    eng.generate(D, 0, 42, 1.0, 2, 0, n, p)
    plan = ReductionPlan(plan_partitions(n, chunk))
    sc = DatasetSchema.generic(p, False)
    for flags in (0, 2):
        eng.dataset_suffstats(D, sc, plan, flags=flags)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.dataset_suffstats(D, sc, plan, flags=flags)
        dt = time.perf_counter() - t0
        print(f"n={n} p={p} chunk={chunk} flags={flags}: {dt * 1e3:.2f} ms, {n / dt:.3g} rows/s", flush=True)
    del D
    torch.cuda.empty_cache()
