# K1w load depth A/B: U = 2 / 3 / 4 k-steps in flight (SSTAT_K1W_U) at every K1w instance
for u in 2 3 4; do
  echo "== U=$u"; SSTAT_K1W_U=$u SWEEP_P=${SWEEP_P:-65,72,73,80,81,88,89,104,105,112,113,120,128} timeout 400 python tools/p_sweep.py 8e9 2>&1
done > gpurun_out/k1w_u.log
