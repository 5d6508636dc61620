# K2 window rule confirmation: defaults at p = 130-200 and the wide-p parity tests
SWEEP_P=130,136,144,152,160,168,176,184,192,200,208 timeout 300 python tools/p_sweep.py 8e9 > gpurun_out/k2_window.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "wide_p or widest or c5_scale or concurrent or buffer_growth" > gpurun_out/k2_window_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k2_window_pytest.log
