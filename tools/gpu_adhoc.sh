for v in "SSTAT_WIDEP_WG=1" "SSTAT_WIDEP_WG=1 SSTAT_WIDEP_NOCLUSTER=1" "SSTAT_WIDEP_WG=1 SSTAT_WIDEP_MAXCLUSTER=2"; do
echo "== $v" >> gpurun_out/wgnc.log
env $v SWEEP_P=192,256,512,1024 timeout 900 python tools/p_sweep.py 2e10 >> gpurun_out/wgnc.log 2>&1
done
