for p in 72 96 128 200 256 300 512 520 1024 2048; do python - <<PY 2>&1 | grep k_widep >> gpurun_out/plans.log
import os; os.environ["SSTAT_DEBUG"]="1"
import torch, paper_2604_23826_b200 as s
e = s.Engine(0); n = 70000; p = $p
D = torch.empty((n, p), dtype=torch.float64, device="cuda"); e.generate(D, 2, 1, 1.0, 0, 0, n, p)
e.dataset_suffstats(D, s.DatasetSchema.generic(p, False), s.ReductionPlan(s.plan_partitions(n, 1 << 20)))
PY
done
timeout 900 python -m pytest tests -q -m gpu -x -k "wide or generated or kats or sharded or c5" 2>&1 | tail -8 > gpurun_out/pytest_wide.log
SSTAT_DEBUG=1 timeout 300 python bench.py --steps 5 --warmup 3 --config c5 --no-cpu --no-e2e > gpurun_out/bench_c5_auto.log 2>&1
