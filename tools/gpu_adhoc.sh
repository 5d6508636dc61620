timeout 300 python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/san_$tool.log
done
