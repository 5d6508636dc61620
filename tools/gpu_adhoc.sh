timeout 900 python bench.py > gpurun_out/bench_default_200.log 2>&1
