# ncu --set full of K1 at C1 (1e6 x 9, one range, 512-row tiles)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_smallp -s 3 -c 1 -o gpurun_out/prof_k1_c1 -f python tools/step_time.py 5 > gpurun_out/prof_k1_c1.log 2>&1
