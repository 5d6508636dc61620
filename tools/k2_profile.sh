# ncu --set full of K2's clustered launch at p = 256 (the idle-slot side launch disabled so the
# capture picks the clustered one); plain timing first
python tools/one_case.py 256 1e7 2 > gpurun_out/k2_plain.log 2>&1
SSTAT_WIDEP_SPARE=0 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_widep_wg -s 1 -c 1 -o gpurun_out/k2_r02 -f python tools/one_case.py 256 1e7 3 > gpurun_out/k2_ncu.log 2>&1
