# K1w W = 8 (one row group per CTA) at 128 < p <= 192 vs K2
{ echo "== K2"; SWEEP_P=136,144,152,160,176,192 timeout 300 python tools/p_sweep.py 8e9 2>&1
echo "== K1w W=8"; SSTAT_SPLITP_MAXP=192 SWEEP_P=136,144,152,160,176,192 timeout 300 python tools/p_sweep.py 8e9 2>&1; } > gpurun_out/k1w_w8.log
SSTAT_SPLITP_MAXP=192 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "wide_p_shapes or k1w_load" > gpurun_out/k1w_w8_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k1w_w8_pytest.log
