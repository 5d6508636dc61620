# Generic gpurun payload: tests + smoke + bench (C2) + optional extra bench configs.
python -m pytest tests -q -m gpu -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.log; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for c in ${EXTRA:-}; do
  timeout 900 python bench.py --steps 5 --warmup 3 --config $c --no-cpu > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?" >> gpurun_out/bench_$c.log
done
