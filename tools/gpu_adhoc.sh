timeout 1200 python -m pytest tests -q -m gpu -x -k "every_p or misaligned or generated or kats" 2>&1 | tail -3 > gpurun_out/pytest_mid.log
SSTAT_DEBUG=1 timeout 900 python tools/p_sweep.py > gpurun_out/p_sweep.log 2>&1
