"""Per-phase time of a dataset_suffstats step (C2, HBM-resident): device step time from
stream events around K back-to-back calls (as bench.py), the library's own event timings
(K1 / folds) and the host wall time per call.  Usage: python tools/step_profile.py [rows] [p]"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
p = int(sys.argv[2]) if len(sys.argv) > 2 else 16
eng = Engine(0)
eng.collect_timings = True
stream = torch.cuda.current_stream()
eng.set_stream(stream.cuda_stream)
D = torch.empty((n, p), dtype=torch.float64, device="cuda")
eng.generate(D, 0, 42, 1.0, 2, 0, n, p)
plan = ReductionPlan(plan_partitions(n, 1 << 20))
schema = DatasetSchema.generic(p, False)
for _ in range(5):
    eng.dataset_suffstats(D, schema, plan)
torch.cuda.synchronize()
K = int(os.environ.get("STEPS", "50"))
kern, fold, total, host = [], [], [], []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(K):
    t0 = time.perf_counter()
    eng.dataset_suffstats(D, schema, plan)
    host.append(time.perf_counter() - t0)
    t = eng.last_timings
    kern.append(t.kernel_seconds)
    fold.append(t.fold_seconds)
    total.append(t.total_seconds)
e1.record(stream)
torch.cuda.synchronize()
dev = e0.elapsed_time(e1) / K * 1e-3
# per-call device interval (event before the call -> event after it) and the gap to the next call
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
for a, b in ev:
    a.record(stream)
    eng.dataset_suffstats(D, schema, plan)
    b.record(stream)
torch.cuda.synchronize()
inside = statistics.mean(a.elapsed_time(b) for a, b in ev) * 1e3
gap = statistics.mean(ev[i][1].elapsed_time(ev[i + 1][0]) for i in range(K - 1)) * 1e3
print(f"  per call on the device {inside:.1f} us (enqueue -> result copied), between calls {gap:.1f} us")
us = lambda v: f"{statistics.mean(v) * 1e6:8.1f} us"  # noqa: E731
print(f"rows={n} p={p}  device step {dev * 1e6:8.1f} us | K1 {us(kern)} | folds {us(fold)} | "
      f"library total {us(total)} | python call {us(host)} | device - K1 - folds "
      f"{(dev - statistics.mean(kern) - statistics.mean(fold)) * 1e6:.1f} us")
