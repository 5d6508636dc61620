timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "every_p or c1 or kats or table1 or generated or misaligned or sharded or streaming" > gpurun_out/x1_pytest.log 2>&1
for v in "SSTAT_K1_NO_X1=1" "X=0"; do
echo "== $v" >> gpurun_out/x1.log
env $v SWEEP_P=9,17 timeout 300 python tools/p_sweep.py 1.6e10 >> gpurun_out/x1.log 2>&1
env $v timeout 300 python tools/step_profile.py 1e6 9 >> gpurun_out/x1.log 2>&1
done
