# K1w at NB = 12: p = 97 by the 12-block-row extra-column split vs the 13-block-row split (SSTAT_K1W_NO_X1), U = 2 / 3 / 4; defaults at p = 90-97
{ for u in 2 3 4; do echo "== x1 U=$u"; SSTAT_K1W_U=$u SWEEP_P=97 timeout 200 python tools/p_sweep.py 8e9 2>&1; done
echo "== no-x1 (NB=13, default U)"; SSTAT_K1W_NO_X1=1 SWEEP_P=97 timeout 200 python tools/p_sweep.py 8e9 2>&1
echo "== defaults"; SWEEP_P=89,90,92,94,96,97 timeout 300 python tools/p_sweep.py 8e9 2>&1; } > gpurun_out/k1w_nb12b.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "k1w or wide_p_shapes or every_p or schedule or concurrent or c5_scale" > gpurun_out/k1w_nb12_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k1w_nb12_pytest.log
