timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
