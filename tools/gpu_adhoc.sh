timeout 600 python tools/refexact_probe.py > gpurun_out/refx_tma16.log 2>&1
