# K1w defaults: parity + the chosen U per width
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "k1w or every_p or wide_p_shapes or misaligned or concurrent or schedule" > gpurun_out/k1w_confirm_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k1w_confirm_pytest.log
SWEEP_P=65,72,73,80,88,89,96,97,104,105,112,120,128 timeout 400 python tools/p_sweep.py 8e9 > gpurun_out/k1w_confirm.log 2>&1
