for v in "SSTAT_WIDEP_WG=1" "SSTAT_WIDEP_WG=1 SSTAT_WIDEP_SROWS=16" "SSTAT_WIDEP_WG=1 SSTAT_WIDEP_SROWS=16 SSTAT_WIDEP_RING=4"; do
echo "== $v" >> gpurun_out/s16.log
env $v SWEEP_P=232,256 timeout 900 python tools/p_sweep.py 4e10 >> gpurun_out/s16.log 2>&1
done
