timeout 1500 python -m pytest tests -q -m gpu -x -k "every_p or generated or kats or c2 or c1 or misaligned or shapes" 2>&1 | tail -3 > gpurun_out/pytest_k1.log
timeout 900 python tools/p_sweep.py > gpurun_out/p_sweep.log 2>&1
