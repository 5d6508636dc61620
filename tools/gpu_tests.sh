# GPU check: box info, smoke, the new / previously failing tests, default bench
(nproc; free -g; df -h /dev/shm; nvidia-smi --query-gpu=name,memory.total --format=csv) > gpurun_out/box.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -q -m gpu -k "group or stream_ordering or pieces or reader or slot or comoments_pair" 2>&1 | tail -40 > gpurun_out/pt_new.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
