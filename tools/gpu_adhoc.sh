start=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "took $(( $(date +%s) - start )) s" >> gpurun_out/bench_default.log
