set -x
nvidia-smi -L
which compute-sanitizer; compute-sanitizer --version
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --target-processes all python tools/sanitize_cases.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_rc.log
done
