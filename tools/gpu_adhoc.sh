run() { tag=$1; shift; env "$@" SSTAT_DEBUG=1 timeout 300 python bench.py --steps 5 --warmup 3 --config c5 --no-cpu --no-e2e > gpurun_out/bench_c5_$tag.log 2>&1; }
run base
run persm1r6 SSTAT_WIDEP_PERSM=1 SSTAT_WIDEP_RING=6
run persm1s8r12 SSTAT_WIDEP_PERSM=1 SSTAT_WIDEP_RING=12 SSTAT_WIDEP_SROWS=8
run c8persm1r6 SSTAT_WIDEP_CONSUMERS=8 SSTAT_WIDEP_RING=6
