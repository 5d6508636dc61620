# Round profiles (1 B200): step times + read floor, the headline's ncu launch list, full captures of
# K1 (C2) and K2 (C5 shard, the clustered launch; NO_K2=1 skips it), and the C1 launch list.  Outputs in gpurun_out/.
python tools/step_time.py 200 > gpurun_out/prof_step_time.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-next --no-c1 --no-c3 --no-c4"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof_launches_c2.csv $B --no-c5 > gpurun_out/prof_launches_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_smallp -s 2 -c 1 \
    -o gpurun_out/prof_k1_c2 -f $B --no-c5 > gpurun_out/prof_k1.log 2>&1
[ -n "$NO_K2" ] || SSTAT_WIDEP_SPARE=0 timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_widep -s 1 -c 1 \
    -o gpurun_out/prof_k2_c5 -f $B > gpurun_out/prof_k2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/prof_launches_c1.csv python tools/step_time.py 3 > gpurun_out/prof_launches_c1.log 2>&1
echo done > gpurun_out/prof_done.log
