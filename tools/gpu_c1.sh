python tools/step_time.py 200 > gpurun_out/step_time.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/c1_launches.csv python tools/step_time.py 3 > gpurun_out/c1_ncu.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/pt_all.log
