timeout 900 python -m pytest tests -q -m gpu -x -k "wide or every_p or widest or c5 or comoments_wide or smoke" 2>&1 | tail -2 > gpurun_out/pytest_wide.log
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --config c5 --no-cpu --no-e2e --no-next > gpurun_out/bench_c5_$i.log 2>&1; done
