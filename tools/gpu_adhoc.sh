timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 python tools/step_profile.py 1e6 9 > gpurun_out/step_c1.log 2>&1
timeout 600 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu --no-e2e --no-next > gpurun_out/bench_c1q.log 2>&1
timeout 600 python bench.py --no-cpu --no-e2e --no-next > gpurun_out/bench_c2q.log 2>&1
