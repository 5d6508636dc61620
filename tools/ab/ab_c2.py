"""C2 K1 A/B between trees, interleaved per rep: python tools/ab/ab_c2.py K REPS tree..."""
import importlib, os, sys
import torch
K, REPS, trees = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3:]
mods = {}
for t in trees:
    for k in [k for k in sys.modules if k.startswith("paper_2604_23826_b200")]:
        del sys.modules[k]
    sys.path.insert(0, os.path.abspath(t))
    mods[t] = importlib.import_module("paper_2604_23826_b200")
    sys.path.pop(0)
n, p = 100_000_000, 16
s = torch.cuda.current_stream()
D = torch.empty((n, p), dtype=torch.float64, device="cuda")
engs = {}
for t in trees:
    e = mods[t].Engine(0)
    e.set_stream(s.cuda_stream)
    e.collect_timings = True
    engs[t] = e
engs[trees[0]].generate(D, 0, 42, 1.0, 2, 0, n, p)
res = {t: [] for t in trees}
for rep in range(REPS):
    for t in (trees if rep % 2 == 0 else trees[::-1]):
        m, e = mods[t], engs[t]
        plan = m.ReductionPlan(m.plan_partitions(n, 1 << 20))
        sc = m.DatasetSchema.generic(p, False)
        for _ in range(3):
            e.dataset_suffstats(D, sc, plan)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ks = []
        a.record(s)
        for _ in range(K):
            e.dataset_suffstats(D, sc, plan)
            ks.append(e.last_timings.kernel_seconds)
        b.record(s)
        torch.cuda.synchronize()
        res[t].append((a.elapsed_time(b) / K * 1e3, sorted(ks)[len(ks) // 2] * 1e6))
        print(f"rep {rep} {t:10s} step {res[t][-1][0]:7.1f} us  K1 {res[t][-1][1]:7.1f} us", flush=True)
for t in trees:
    st = sorted(x[0] for x in res[t]); k1 = sorted(x[1] for x in res[t])
    print(f"{t:10s} median step {st[len(st) // 2]:7.1f} us  K1 {k1[len(k1) // 2]:7.1f} us  ({12.8e9 / (k1[len(k1) // 2] * 1e-6) / 1e9:.0f} GB/s)")
