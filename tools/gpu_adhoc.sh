timeout 1500 python -m pytest tests -q -m gpu -x -k "wide or every_p or widest or comoments_wide or smoke or c5" 2>&1 | tail -3 > gpurun_out/pytest_wide.log
SWEEP_P=96,136,160,192,256,384,512 timeout 900 python tools/p_sweep.py > gpurun_out/p_sweep_sums.log 2>&1
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --config c5 --no-cpu --no-e2e --no-next > gpurun_out/bench_c5_$i.log 2>&1; done
