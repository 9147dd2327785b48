mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  echo "=== $tool"
  timeout 900 compute-sanitizer --tool $tool --target-processes all python scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
