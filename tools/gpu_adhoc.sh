timeout 1500 python -m pytest tests -q -m gpu -x -k "wide or every_p or widest or comoments_wide or smoke" 2>&1 | tail -3 > gpurun_out/pytest_wide.log
SSTAT_DEBUG=1 timeout 1200 python tools/p_sweep.py > gpurun_out/p_sweep.log 2>&1
