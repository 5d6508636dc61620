timeout 600 python -m pytest tests -q -m gpu -x -k "feeder or streaming" 2>&1 | tail -3 > gpurun_out/pytest_feeder.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/bench_default.log
