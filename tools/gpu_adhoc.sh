timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c5_full.log 2>&1
timeout 600 python bench.py --impl reference --config c5 --steps 2 --warmup 1 > gpurun_out/bench_c5_ref.log 2>&1
timeout 600 python bench.py --config c1 --steps 20 --warmup 3 > gpurun_out/bench_c1_full.log 2>&1
