timeout 900 python -m pytest tests -q -m gpu -x -k "concurrent" 2>&1 | tail -15 > gpurun_out/pytest_conc.log
