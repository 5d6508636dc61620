# Round check on one B200: smoke, the whole -m gpu suite, the default bench and its reference arm,
# C1/C2 step times.  Outputs in gpurun_out/.
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu --durations=10 2>&1 | tail -40 > gpurun_out/pt_all.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
python tools/step_time.py 200 > gpurun_out/step_time.log 2>&1
SSTAT_WIDEP_SPARE=0 timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_widep -s 1 -c 1 \
    -o gpurun_out/prof_k2b_c5 -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-next --no-c1 --no-c3 --no-c4 > gpurun_out/prof_k2b.log 2>&1
