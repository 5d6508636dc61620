export SWEEP_P=96,128,192,256,384,512
for v in "SSTAT_WIDEP_PF=0" "SSTAT_WIDEP_PF=4" "SSTAT_WIDEP_PF=8" "SSTAT_WIDEP_PF=16" "SSTAT_WIDEP_PF=32"; do
  echo "== $v" >> gpurun_out/pf.log
  env $v SSTAT_SPLITP=0 timeout 300 python tools/p_sweep.py 1.6e10 >> gpurun_out/pf.log 2>&1
done
timeout 900 python bench.py --config c5 --no-cpu --no-e2e --no-next > gpurun_out/bench_c5_pf.log 2>&1
