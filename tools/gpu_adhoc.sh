timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
SSTAT_DEBUG=1 timeout 900 python tools/p_sweep.py > gpurun_out/p_sweep.log 2>&1
