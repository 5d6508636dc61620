for v in 8 16; do echo "== SROWS=$v"; SSTAT_WIDEP_SROWS=$v SWEEP_P=256 timeout 600 python tools/ab/p_sweep_tree.py . 1e11; done > gpurun_out/k2_srows.log 2>&1
