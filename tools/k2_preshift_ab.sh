# The pre-shift A/B of profiles/r02_k2_preshift_ab.log (ab/nopre: the package tree without the pre-shift change)
TREE=ab/nopre WIDTHS=256,248,512 BYTES=1e11 bash tools/k2_ab.sh > gpurun_out/k2_pre.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x -k "wide_p or c5 or p256 or schedule or group_wide or comoments_wide or widest or concurrent" 2>&1 | tail -3 > gpurun_out/k2_pre_tests.log
