timeout 900 python -m pytest tests -q -m gpu -x -k "every_p or widest or schedule" 2>&1 | tail -15 > gpurun_out/pytest_new.log
