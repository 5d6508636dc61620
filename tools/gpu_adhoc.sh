timeout 600 python tools/register_probe.py 8 > gpurun_out/register_probe.log 2>&1
