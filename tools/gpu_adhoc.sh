timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "every_p or c1 or kats or table1 or generated or misaligned or sharded or streaming" > gpurun_out/x1_pytest.log 2>&1
