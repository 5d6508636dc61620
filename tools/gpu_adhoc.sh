for v in "SSTAT_WIDEP_WG=1 SSTAT_WIDEP_DBG=3" "SSTAT_WIDEP_WG=1 SSTAT_WIDEP_DBG=3 SSTAT_WIDEP_SROWS=8"; do
echo "== $v" >> gpurun_out/shiftdbg3.log
env $v SWEEP_P=256,512 timeout 900 python tools/p_sweep.py 1.6e10 >> gpurun_out/shiftdbg3.log 2>&1
done
