"""C2 (or C1) step with and without the library's timing events, alternated to cancel clock drift:
    python tools/onoff.py [ROUNDS] [K] [c1]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions  # noqa: E402

ROUNDS = int(sys.argv[1]) if len(sys.argv) > 1 else 6
K = int(sys.argv[2]) if len(sys.argv) > 2 else 50
C1 = len(sys.argv) > 3 and sys.argv[3] == "c1"
n, p, kind, n_int = (1_000_000, 9, 1, 0) if C1 else (100_000_000, 16, 0, 2)
eng = Engine(0)
s = torch.cuda.current_stream()
eng.set_stream(s.cuda_stream)
D = torch.empty((n, p), dtype=torch.float64, device="cuda")
eng.generate(D, kind, 42, 1.0, n_int, 0, n, p)
plan = ReductionPlan(plan_partitions(n, 1 << 20))
sc = DatasetSchema.generic(p, C1)
acc = {True: [], False: []}
for r in range(ROUNDS):
    for timed in ((True, False) if r % 2 == 0 else (False, True)):
        eng.collect_timings = timed
        for _ in range(3):
            eng.dataset_suffstats(D, sc, plan)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(K):
            eng.dataset_suffstats(D, sc, plan)
        b.record(s)
        torch.cuda.synchronize()
        acc[timed].append(a.elapsed_time(b) / K * 1e3)
        print(f"round {r} timings={'on ' if timed else 'off'} step {acc[timed][-1]:.1f} us", flush=True)
for timed in (True, False):
    v = sorted(acc[timed])
    print(f"timings={'on ' if timed else 'off'} median {v[len(v) // 2]:.1f} us min {v[0]:.1f} us")
