timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "misaligned" > gpurun_out/mis_pytest.log 2>&1
