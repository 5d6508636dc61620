"""K1 A/B over sizes and widths between trees, interleaved per rep: python tools/ab/ab_sizes.py REPS tree..."""
import importlib, os, sys
import torch
REPS, trees = int(sys.argv[1]), sys.argv[2:]
mods = {}
for t in trees:
    for k in [k for k in sys.modules if k.startswith("paper_2604_23826_b200")]:
        del sys.modules[k]
    sys.path.insert(0, os.path.abspath(t))
    mods[t] = importlib.import_module("paper_2604_23826_b200")
    sys.path.pop(0)
CASES = [(10_000_000, 16), (20_000_000, 16), (50_000_000, 16), (100_000_000, 16), (500_000_000, 16),
         (100_000_000, 9), (100_000_000, 8), (50_000_000, 32), (25_000_000, 64), (40_000_000, 24)]
s = torch.cuda.current_stream()
engs = {}
for t in trees:
    e = mods[t].Engine(0)
    e.set_stream(s.cuda_stream)
    e.collect_timings = True
    engs[t] = e
for n, p in CASES:
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engs[trees[0]].generate(D, 0, 42, 1.0, 2, 0, n, p)
    K = max(3, int(2e10 / (n * p * 8)))
    res = {t: [] for t in trees}
    for rep in range(REPS):
        for t in (trees if rep % 2 == 0 else trees[::-1]):
            m, e = mods[t], engs[t]
            plan = m.ReductionPlan(m.plan_partitions(n, 1 << 20))
            sc = m.DatasetSchema.generic(p, False)
            for _ in range(2):
                e.dataset_suffstats(D, sc, plan)
            ks = []
            for _ in range(K):
                e.dataset_suffstats(D, sc, plan)
                ks.append(e.last_timings.kernel_seconds)
            res[t].append(sorted(ks)[len(ks) // 2])
    line = f"n={n:.0e} p={p:3d}"
    for t in trees:
        v = sorted(res[t])[len(res[t]) // 2]
        line += f" | {t}: {v * 1e6:8.1f} us {n * p * 8 / v / 1e9:5.0f} GB/s"
    print(line, flush=True)
    del D
    torch.cuda.empty_cache()
