set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
lscpu | head -20; nproc; free -g; df -h /tmp /dev/shm /root
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/probe/fp64_probe 2>&1 | tee gpurun_out/probe.log
kill $SMI
