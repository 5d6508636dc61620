for i in 1 2; do
  echo "== balanced (default)"; SWEEP_P=256,248,512,1024 timeout 600 python tools/p_sweep.py 1e11 2>&1 | python -c "import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['p'], round(d['fp64_tf_per_s'],2), 'TF/s', round(d['kernel_ms'],2), 'ms')
    except Exception: print(l.rstrip())"
  echo "== SSTAT_WIDEP_NOBALANCE=1"; SSTAT_WIDEP_NOBALANCE=1 SWEEP_P=256,248 timeout 600 python tools/p_sweep.py 1e11 2>&1 | python -c "import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['p'], round(d['fp64_tf_per_s'],2), 'TF/s', round(d['kernel_ms'],2), 'ms')
    except Exception: print(l.rstrip())"
done > gpurun_out/k2_bal.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x -k "wide_p or c5 or p256 or schedule or group_wide or smoke or comoments_wide or widest or concurrent" 2>&1 | tail -5 > gpurun_out/k2_bal_tests.log
