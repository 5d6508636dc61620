"""Throughput of the accumulate kernels across widths p (HBM-resident, 2^20-row ranges):
rows/s, HBM GB/s and FP64 TF/s of the K1/K2 launch (library events), for the roofline
crossover between the HBM-bound and the DMMA-bound regimes.
    python tools/p_sweep.py [bytes_per_case]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 8e9
eng = Engine(0)
eng.collect_timings = True
for p in [int(x) for x in os.environ.get("SWEEP_P", "8,16,24,32,40,48,56,64,65,72,80,96,104,112,120,128,192,256,384,512").split(",")]:
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
    print(json.dumps({"p": p, "rows": n, "kernel_ms": k * 1e3, "rows_per_s": n / k, "hbm_gb_per_s": n * p * 8 / k / 1e9,
                      "fp64_tf_per_s": n * p * (p + 2) / k / 1e12}), flush=True)
    del D
    torch.cuda.empty_cache()
