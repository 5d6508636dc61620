for i in 1 2; do python ab/ab_step.py ab/r1 100; python ab/ab_step.py . 100; done > gpurun_out/ab.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -c 12 --csv --log-file gpurun_out/c2_launches_r2.csv python ab/ab_step.py . 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -c 12 --csv --log-file gpurun_out/c2_launches_r1.csv python ab/ab_step.py ab/r1 1 > /dev/null 2>&1
