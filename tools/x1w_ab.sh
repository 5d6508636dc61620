# K1w extra-column variant: parity tests, then A/B widths p = 8 NB + 1 (x1 vs SSTAT_K1W_NO_X1)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "k1w or every_p or wide_p_shapes or misaligned or concurrent" > gpurun_out/x1w_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/x1w_pytest.log
SWEEP_P=65,73,81,89,97,105,113,121,72,128 timeout 600 python tools/p_sweep.py 8e9 > gpurun_out/x1w_on.log 2>&1
SSTAT_K1W_NO_X1=1 SWEEP_P=65,73,81,89,97,105,113,121 timeout 600 python tools/p_sweep.py 8e9 > gpurun_out/x1w_off.log 2>&1
