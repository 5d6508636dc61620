for p in 384 512 1024; do
  for c in 8 4; do SSTAT_DEBUG=1 SSTAT_WIDEP_CONSUMERS=$c timeout 300 python tools/one_case.py $p $(( 8000000000 / (8 * p) )) 3 2>&1 | grep -E "k_widep|^$p" | tail -2 | sed "s/^/C=$c /"; done
done > gpurun_out/wide_c.log 2>&1
