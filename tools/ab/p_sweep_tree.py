"""K1/K2 kernel time across widths for one package tree (A/B between trees):
    SWEEP_P=256,136 python tools/ab/p_sweep_tree.py <tree> [bytes_per_case]
Prints "p TF/s ms" per width (library events, best of 3 after 2 warm-ups)."""
import os
import sys

tree = sys.argv[1]
sys.path.insert(0, os.path.abspath(tree))
import torch  # noqa: E402

from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions  # noqa: E402

budget = float(sys.argv[2]) if len(sys.argv) > 2 else 5e10
eng = Engine(0)
eng.collect_timings = True
for p in [int(x) for x in os.environ.get("SWEEP_P", "256").split(",")]:
    n = int(budget // (8 * p))
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    eng.generate(D, 2, 1, 1.0, 0, 0, n, p)
    plan = ReductionPlan(plan_partitions(n, 1 << 20))
    schema = DatasetSchema.generic(p, False)
    for _ in range(2):
        eng.dataset_suffstats(D, schema, plan)
    ks = []
    for _ in range(3):
        eng.dataset_suffstats(D, schema, plan)
        ks.append(eng.last_timings.kernel_seconds)
    k = min(ks)
    print(f"{p} {n * p * (p + 2) / k / 1e12:.2f} TF/s {k * 1e3:.2f} ms", flush=True)
    del D
    torch.cuda.empty_cache()
