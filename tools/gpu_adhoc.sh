for i in 1 2; do timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3 >> gpurun_out/pytest_rep.log; done
timeout 600 python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo "rc=$?" >> gpurun_out/san_plain.log
