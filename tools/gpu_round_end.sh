# round-end confirmation: full GPU suite, smoke, default bench, width sweep
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -5 > gpurun_out/re_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/re_smoke.log
timeout 900 python bench.py > gpurun_out/re_bench_default.log 2>&1
SWEEP_P=8,16,24,32,40,48,56,64,65,72,80,89,92,96,97,104,112,120,128,136,144,160,192,256,384,512 timeout 900 python tools/p_sweep.py 8e9 > gpurun_out/re_p_sweep.log 2>&1
