timeout 900 python -m pytest tests -q -m gpu -x -k "comoments or glue" 2>&1 | tail -3 > gpurun_out/pytest_cm.log
timeout 600 python bench.py --steps 5 --warmup 3 --config c5 --no-cpu --no-e2e > gpurun_out/bench_c5_cm.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c2_cm.log 2>&1
