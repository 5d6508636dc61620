timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_widep -s 1 -c 1 \
    -o gpurun_out/k2_full -f python bench.py --steps 1 --warmup 3 --config c5 --no-cpu --no-e2e > gpurun_out/ncu_k2.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_k2.log
