# K2 around the measured window: default vs the 4-warp kernel with 3x3 / 4x4 rectangles
{ for cfg in default "0 3" "0 4"; do
  if [ "$cfg" = default ]; then echo "== default"; SWEEP_P=130,144,168,184,192,200 timeout 200 python tools/p_sweep.py 8e9 2>&1;
  else set -- $cfg; echo "== WG=$1 R=$2"; SSTAT_WIDEP_WG=$1 SSTAT_WIDEP_R=$2 SWEEP_P=130,144,168,184,192,200 timeout 200 python tools/p_sweep.py 8e9 2>&1; fi
done; } > gpurun_out/k2_r_sweep2.log
