timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x -k "wide or widest or misaligned or c5 or comoments" > gpurun_out/wide_pytest.log 2>&1
