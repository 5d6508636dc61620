# K1 load depth A/B at the one-CTA-per-SM widths: default U = 4 vs SSTAT_K1_U = 6 / 8
for u in 0 6 8; do
  if [ $u = 0 ]; then unset SSTAT_K1_U; else export SSTAT_K1_U=$u; fi
  echo "== U=$u"; SWEEP_P=${SWEEP_P:-41,44,48,49,52,56} timeout 300 python tools/p_sweep.py 8e9 2>&1
done > gpurun_out/k1_u.log
unset SSTAT_K1_U
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "k1_load_depth" > gpurun_out/k1_u_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k1_u_pytest.log
