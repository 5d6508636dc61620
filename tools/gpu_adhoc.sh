timeout 900 python bench.py --steps 5 --warmup 3 --config c5 > gpurun_out/bench_c5.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -x -k "wide_p_schedule or c5 or comoments_wide" 2>&1 | tail -2 > gpurun_out/pytest_new.log
