timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
SWEEP_P=96,136,168,200,232,256,296,352,384,416,448,512,640,768,1024,2048 SSTAT_DEBUG=1 timeout 900 python tools/p_sweep.py 4e10 > gpurun_out/sweep_new.log 2>&1
timeout 600 python bench.py --config c5 --no-cpu --no-e2e --no-next > gpurun_out/bench_c5_wg.log 2>&1
