# The K2 ceiling experiments of profiles/r02_k2_ceiling_experiments.log (ab/nowait, ab/nowaitdexp_norelease: one-change copies of the package tree, see the log)
for t in . ab/nowait ab/nowaitdexp_norelease; do echo "== $t"; SWEEP_P=256 timeout 300 python tools/ab/p_sweep_tree.py $t 1e11; done > gpurun_out/k2_exp.log 2>&1
