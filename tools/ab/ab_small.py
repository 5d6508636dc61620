"""Small-plan K1 A/B between package trees: python tools/ab/ab_small.py <tree> [<tree> ...]
Per case: K1 (library events) median and the untimed step, trees interleaved per rep."""
import importlib
import os
import sys

import torch

trees = sys.argv[1:]
CASES = [("C1 p9x1", 1_000_000, 9, 1, 0), ("p16 1e6", 1_000_000, 16, 0, 2), ("p16 4e6", 4_000_000, 16, 0, 2),
         ("p17 2e6", 2_000_000, 17, 0, 0), ("p8 2e6", 2_000_000, 8, 0, 0), ("p12 2e6", 2_000_000, 12, 0, 0)]
mods = {}
for t in trees:
    for k in [k for k in sys.modules if k.startswith("paper_2604_23826_b200")]:
        del sys.modules[k]
    sys.path.insert(0, os.path.abspath(t))
    mods[t] = importlib.import_module("paper_2604_23826_b200")
    sys.path.pop(0)
K = 300
s = torch.cuda.current_stream()
for name, n, p, kind, n_int in CASES:
    res = {t: ([], []) for t in trees}
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engs = {}
    for t in trees:
        m = mods[t]
        e = m.Engine(0)
        e.set_stream(s.cuda_stream)
        engs[t] = (m, e)
    engs[trees[0]][1].generate(D, kind, 42, 1.0, n_int, 0, n, p)
    ref = None
    for rep in range(4):
        for t in trees:
            m, e = engs[t]
            plan = m.ReductionPlan(m.plan_partitions(n, 1 << 20))
            sc = m.DatasetSchema.generic(p, kind == 1)
            e.collect_timings = True
            ks = []
            for _ in range(K // 3):
                r = e.dataset_suffstats(D, sc, plan)
                ks.append(e.last_timings.kernel_seconds * 1e6)
            b = (r.sums.tobytes(), r.cross.tobytes())
            if ref is None:
                ref = b
            assert b == ref, (name, t, "result bits differ")
            e.collect_timings = False
            for _ in range(5):
                e.dataset_suffstats(D, sc, plan)
            torch.cuda.synchronize()
            a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(K):
                e.dataset_suffstats(D, sc, plan)
            bb.record(s)
            torch.cuda.synchronize()
            ks.sort()
            res[t][0].append(ks[len(ks) // 2])
            res[t][1].append(a.elapsed_time(bb) / K * 1e3)
    for t in trees:
        k1 = sorted(res[t][0])[len(res[t][0]) // 2]
        st = sorted(res[t][1])[len(res[t][1]) // 2]
        print(f"{name:10s} {t:10s} K1 {k1:7.1f} us ({n * p * 8 / k1 / 1e6:5.2f} TB/s)  step {st:7.1f} us", flush=True)
    for t in trees:
        engs[t][1].close()
    del D
    torch.cuda.empty_cache()
