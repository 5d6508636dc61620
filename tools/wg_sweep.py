"""K2 variant sweep: classic 4-warp CTAs vs the 12-consumer-warp k_widep_wg, each with the
rectangle side R = 3 or 4 (and the default choice), FP64 TF/s of the accumulate launch(es) per p.
    SWEEP_P=136,192,... python tools/wg_sweep.py [bytes_per_case]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 4e10
eng = Engine(0)
eng.collect_timings = True
os.environ["SSTAT_SPLITP"] = "0"
for p in [int(x) for x in os.environ.get("SWEEP_P", "136,192,256,384,512").split(",")]:
    n = int(budget // (8 * p))
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    eng.generate(D, 2, 1, 1.0, 0, 0, n, p)
    plan = ReductionPlan(plan_partitions(n, 1 << 20))
    schema = DatasetSchema.generic(p, False)
    row = {"p": p}
    for wg, R in (("0", "0"), ("0", "3"), ("0", "4"), ("1", "3"), ("1", "4")):
        if True:
            os.environ["SSTAT_WIDEP_WG"] = wg
            if R == "0":
                os.environ.pop("SSTAT_WIDEP_R", None)
            else:
                os.environ["SSTAT_WIDEP_R"] = R
            eng.dataset_suffstats(D, schema, plan)
            ks = []
            for _ in range(3):
                eng.dataset_suffstats(D, schema, plan)
                ks.append(eng.last_timings.kernel_seconds)
            row[f"wg{wg}_R{R}"] = round(n * p * (p + 2) / min(ks) / 1e12, 2)
    print(json.dumps(row), flush=True)
    del D
    torch.cuda.empty_cache()
