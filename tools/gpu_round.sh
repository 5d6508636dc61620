# Round check on one B200: smoke, the whole -m gpu suite, the default bench, C1/C2 step times.
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu --durations=15 2>&1 | tail -40 > gpurun_out/pt_all.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python tools/step_time.py 200 > gpurun_out/step_time.log 2>&1
