timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4 > gpurun_out/pytest_gpu.log
timeout 300 python tools/step_profile.py > gpurun_out/step_profile.log 2>&1
timeout 300 python tools/step_profile.py 1e6 9 >> gpurun_out/step_profile.log 2>&1
