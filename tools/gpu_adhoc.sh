SWEEP_P=192,200,232,296,352,384 SSTAT_DEBUG=1 timeout 900 python tools/p_sweep.py 1.6e10 > gpurun_out/rule4.log 2>&1
