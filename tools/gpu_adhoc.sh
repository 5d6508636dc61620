timeout 600 python -m pytest tests -q -m gpu -x -k "checkpoint or sharded" 2>&1 | tail -15 > gpurun_out/pytest_ckpt.log
