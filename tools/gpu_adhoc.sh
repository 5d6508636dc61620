timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 300 python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo "rc=$?" >> gpurun_out/san_plain.log
timeout 600 python bench.py --no-cpu --no-e2e --no-next > gpurun_out/bench_quick.log 2>&1
