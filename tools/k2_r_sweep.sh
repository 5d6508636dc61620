# K2 at the widths whose block count pads badly (p = 136 / 152 / 160 / 176): default plan vs forced kernel x rectangle side
{ echo "== default"; SWEEP_P=136,152,160,176 timeout 200 python tools/p_sweep.py 8e9 2>&1
for wg in 0 1; do for r in 2 3 4; do
  echo "== WG=$wg R=$r"; SSTAT_WIDEP_WG=$wg SSTAT_WIDEP_R=$r SWEEP_P=136,152,160,176 timeout 200 python tools/p_sweep.py 8e9 2>&1
done; done; } > gpurun_out/k2_r_sweep.log
