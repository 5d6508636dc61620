timeout 1500 python -m pytest tests -q -m gpu -x -k "kats or table1 or generated or nonfinite or every_source or glue or c1 or widest or sharded or binary32 or column_sum" 2>&1 | tail -3 > gpurun_out/pytest_ref.log
timeout 600 python tools/refexact_probe.py > gpurun_out/refexact.log 2>&1
