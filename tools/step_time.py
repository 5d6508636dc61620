"""Device-timed dataset_suffstats step at C1 (1e6 x (8 + ID)) and C2 (1e8 x 16), as bench.py
times it (CUDA events around K back-to-back calls on torch's stream), with and without the
timing events, plus the per-call K1 / fold split from the timings.
    python tools/step_time.py [K]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for name, n, p, kind, n_int in (("C1", 1_000_000, 9, 1, 0), ("C2", 100_000_000, 16, 0, 2)):
    eng = Engine(0)
    s = torch.cuda.current_stream()
    eng.set_stream(s.cuda_stream)
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    eng.generate(D, kind, 42, 1.0, n_int, 0, n, p)
    plan = ReductionPlan(plan_partitions(n, 1 << 20))
    sc = DatasetSchema.generic(p, kind == 1)
    for timed in (True, False):
        eng.collect_timings = timed
        for _ in range(5):
            eng.dataset_suffstats(D, sc, plan)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(K):
            eng.dataset_suffstats(D, sc, plan)
        b.record(s)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / K
        extra = ""
        if timed:
            t = eng.last_timings
            extra = f" K1 {t.kernel_seconds * 1e6:.1f} us folds {t.fold_seconds * 1e6:.1f} us kernel {t.kernel.decode()}"
        print(f"{name} timings={'on ' if timed else 'off'} step {ms * 1e3:.1f} us{extra}", flush=True)
    # the practical read floor at this size: a plain device-wide read of the same bytes
    # (torch.sum over the tensor), timed the same way
    for _ in range(5):
        D.sum()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(K):
        D.sum()
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / K
    print(f"{name} read floor (torch.sum of the {n * p * 8 / 1e6:.0f} MB): {ms * 1e3:.1f} us "
          f"= {n * p * 8 / ms / 1e9 * 1e3 / 1e3:.2f} TB/s", flush=True)
    del D
    eng.close()
    torch.cuda.empty_cache()
