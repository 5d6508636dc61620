timeout 900 python -m pytest tests/test_gpu_next.py -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest_new.log
