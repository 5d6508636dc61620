# K2 A/B: this build vs an alternative library (SSTAT_LIB=<ALT>), twice each, at the widths WIDTHS
for i in 1 2; do
  for lib in paper_2604_23826_b200/libsstat_b200.so ${ALT:-ab/cs0/libsstat_b200.so}; do
    echo "== $lib"; SSTAT_LIB=$lib SWEEP_P=${WIDTHS:-256,136,192,512,1024} timeout 600 python tools/p_sweep.py ${BYTES:-2e10} 2>&1 | python -c "import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['p'], round(d['fp64_tf_per_s'],2), 'TF/s', round(d['kernel_ms'],2), 'ms')
    except Exception: print(l.rstrip())"
  done
done
