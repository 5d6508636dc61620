timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 300 python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo "rc=$?" >> gpurun_out/san_plain.log
for g in 0 1; do
  if [ $g = 0 ]; then export SSTAT_NO_GRAPH=1; else unset SSTAT_NO_GRAPH; fi
  timeout 300 python tools/step_profile.py 1e6 9 | sed "s/^/graph=$g /" >> gpurun_out/graph_prof.log 2>&1
  timeout 300 python tools/step_profile.py | sed "s/^/graph=$g /" >> gpurun_out/graph_prof.log 2>&1
  timeout 600 python bench.py --config c1 --no-cpu --no-e2e --no-next | sed "s/^/graph=$g /" >> gpurun_out/graph_bench.log 2>&1
  timeout 600 python bench.py --no-cpu --no-e2e --no-next | sed "s/^/graph=$g /" >> gpurun_out/graph_bench.log 2>&1
done
