"""Reference-order pass (SSTAT_FLAG_REFEXACT) at C2 (1e8 x 16, 96 ranges), HBM-resident: per-call
time and the accumulate kernel's event time.  python tools/ab/refexact_c2.py [tree] [K]"""
import os
import sys

tree = sys.argv[1] if len(sys.argv) > 1 else "."
sys.path.insert(0, os.path.abspath(tree))
import torch  # noqa: E402

from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions  # noqa: E402

K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n, p = 100_000_000, 16
eng = Engine(0)
eng.collect_timings = True
D = torch.empty((n, p), dtype=torch.float64, device="cuda")
eng.generate(D, 0, 42, 1.0, 2, 0, n, p)
plan = ReductionPlan(plan_partitions(n, 1 << 20))
sc = DatasetSchema.generic(p, False)
r0 = eng.dataset_suffstats(D, sc, plan, flags=2)
ks = []
for _ in range(K):
    r = eng.dataset_suffstats(D, sc, plan, flags=2)
    ks.append(eng.last_timings.kernel_seconds)
    assert r.bit_equal(r0)
print(f"{tree}: refexact C2 kernel {min(ks) * 1e3:.2f} ms ({eng.last_timings.kernel.decode()}), "
      f"sha {hash((r0.sums.tobytes(), r0.cross.tobytes())) & 0xffffffff:08x}", flush=True)
