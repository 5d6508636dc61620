# K2 past the window: default vs forced kernel x rectangle side at p = 216-320
{ for cfg in default "0 3" "0 4" "1 3"; do
  if [ "$cfg" = default ]; then echo "== default"; SWEEP_P=216,232,240,264,280,296,320 timeout 200 python tools/p_sweep.py 8e9 2>&1;
  else set -- $cfg; echo "== WG=$1 R=$2"; SSTAT_WIDEP_WG=$1 SSTAT_WIDEP_R=$2 SWEEP_P=216,232,240,264,280,296,320 timeout 200 python tools/p_sweep.py 8e9 2>&1; fi
done; } > gpurun_out/k2_r_sweep3.log
