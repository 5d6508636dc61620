timeout 300 python tools/h2d_probe.py > gpurun_out/h2d.log 2>&1
