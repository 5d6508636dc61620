# Round measurement: tests, smoke, bench (default + configs), ncu launch list and full captures.
set -x
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_reference.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 --config c1 > gpurun_out/bench_c1.log 2>&1
for c in c4 c5; do timeout 900 python bench.py --steps 5 --warmup 3 --config $c > gpurun_out/bench_$c.log 2>&1; done
timeout 900 python bench.py --impl reference --config c5 --steps 2 --warmup 1 > gpurun_out/bench_reference_c5.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-next > gpurun_out/plain.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-next > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_smallp -s 2 -c 1 \
    -o gpurun_out/k1_full -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-next > gpurun_out/ncu_k1.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --config c5 --no-cpu --no-e2e > gpurun_out/plain_c5.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_widep -s 0 -c 1 \
    -o gpurun_out/k2_full -f python bench.py --steps 2 --warmup 3 --config c5 --no-cpu --no-e2e --no-next > gpurun_out/ncu_k2.log 2>&1
echo done
