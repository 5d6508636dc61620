"""Small runs of every device path, with cross-checks (device vs host-staged source bits), for
compute-sanitizer (memcheck / racecheck / synccheck) where it is available — on the round's GPU
pool it is closed, so this runs plain as an all-paths smoke:
K1 (p = 16, 24), K1w (p = 72, 104), K2 (p = 96, 256: clusters, TMA multicast, the idle-slot
side launch), odd-p K2 staging, host-staged sources, reference order (staged and plain),
column_sum, co-moments, the non-finite path.
    compute-sanitizer --tool memcheck python tools/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionError, ReductionPlan, plan_partitions  # noqa: E402


def main():
    eng = Engine(0)
    for p, n, chunk in ((16, 40_000, 9_001), (24, 30_000, 7_001), (72, 40_000, 33_333), (104, 40_000, 33_333),
                        (96, 40_000, 33_333), (256, 70_000, 33_333), (129, 9_000, 4_001)):
        D = torch.empty((n, p), dtype=torch.float64, device="cuda")
        eng.generate(D, 2, 3, 1.0, 0, 0, n, p)
        sc = DatasetSchema.generic(p, False)
        pl = ReductionPlan(plan_partitions(n, chunk))
        a = eng.dataset_suffstats(D, sc, pl)
        b = eng.dataset_suffstats(D.cpu().numpy(), sc, pl)
        assert a.bit_equal(b), p
        if p <= 104:
            eng.dataset_suffstats(D, sc, pl, flags=2)
        eng.comoments(D, sc, pl)
        eng.column_sum(D, 0, pl, p=p)
        print(f"p={p} ok", flush=True)
        del D
    X = np.random.default_rng(1).normal(size=(5_000, 16))
    X[3_333, 5] = np.nan
    try:
        eng.dataset_suffstats(torch.from_numpy(X).cuda(), DatasetSchema.generic(16, False),
                              ReductionPlan(plan_partitions(5_000, 1_000)))
        raise AssertionError("non-finite not reported")
    except ReductionError:
        pass
    eng.close()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
