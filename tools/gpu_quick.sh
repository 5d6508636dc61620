# quick loop: selected tests + selected bench configs (no cpu/e2e)
timeout ${TTIMEOUT:-900} python -m pytest tests -q -m gpu -x ${TESTS:-} 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-c2}; do
  timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 --config $c --no-cpu --no-e2e > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?" >> gpurun_out/bench_$c.log
done
