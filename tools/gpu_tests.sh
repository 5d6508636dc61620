python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x -k "group or stream_ordering or pieces or reader or slot" 2>&1 | tail -30 > gpurun_out/pt_new.log
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -30 > gpurun_out/pt_all.log
