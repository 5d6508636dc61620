"""Cold small-plan calls (L2 flushed by a 256 MB read before every call): per-call device time
and K1 event time for a few shapes.  python tools/ab/cold_calls.py [tree]"""
import os
import sys

tree = sys.argv[1] if len(sys.argv) > 1 else "."
sys.path.insert(0, os.path.abspath(tree))
import torch  # noqa: E402

from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions  # noqa: E402

CASES = [(1_000_000, 9, 1, 1 << 20), (1_000_000, 16, 0, 1 << 20), (2_000_000, 16, 0, 1 << 20),
         (4_000_000, 16, 0, 1 << 20), (2_000_000, 8, 0, 1 << 20), (300_000, 32, 0, 1 << 20),
         (3_000_000, 9, 1, 100_000), (500_000, 24, 0, 1 << 20)]
if os.environ.get("COLD_CASES"):  # n:p:kind:chunk,...
    CASES = [tuple(int(float(v)) for v in c.split(":")) for c in os.environ["COLD_CASES"].split(",")]
eng = Engine(0)
s = torch.cuda.current_stream()
eng.set_stream(s.cuda_stream)
flush = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
tag = os.environ.get("SSTAT_K1_ONEWAVE", "-")
for n, p, kind, chunk in CASES:
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    eng.generate(D, kind, 7, 1.0, 0 if kind else 2, 0, n, p)
    plan = ReductionPlan(plan_partitions(n, chunk))
    sc = DatasetSchema.generic(p, kind == 1)
    out = {}
    for timed in (False, True):
        eng.collect_timings = timed
        ts, ks = [], []
        for it in range(105):
            flush.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            eng.dataset_suffstats(D, sc, plan)
            b.record(s)
            torch.cuda.synchronize()
            if it >= 5:
                ts.append(a.elapsed_time(b) * 1e3)
                if timed:
                    ks.append(eng.last_timings.kernel_seconds * 1e6)
        out[timed] = (sorted(ts)[len(ts) // 2], sorted(ks)[len(ks) // 2] if ks else 0)
    print(f"onewave={tag} n={n:.0e} p={p:2d} chunk={chunk}: call {out[False][0]:6.1f} us  K1(events) {out[True][1]:6.1f} us",
          flush=True)
    del D
    torch.cuda.empty_cache()
