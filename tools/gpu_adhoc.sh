timeout 900 python tools/p_sweep.py > gpurun_out/p_sweep.log 2>&1
