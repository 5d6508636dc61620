timeout 300 python bench.py --steps 2 --warmup 3 --config c5 --no-cpu --no-e2e --no-next > gpurun_out/plain_c5b.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv \
    python bench.py --steps 2 --warmup 3 --config c5 --no-cpu --no-e2e --no-next > gpurun_out/ncu_launch_c5.log 2>&1
