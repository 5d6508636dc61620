timeout 1500 python -m pytest tests -q -m gpu -x -k "wide or every_p or widest or c5 or comoments_wide or misaligned or growth" 2>&1 | tail -3 > gpurun_out/pytest_wide.log
SSTAT_DEBUG=1 timeout 900 python tools/p_sweep.py > gpurun_out/p_sweep.log 2>&1
