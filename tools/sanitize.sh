# compute-sanitizer evidence
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/r2_sanitizer_${TAG:-r2}_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r2_sanitizer_${TAG:-r2}_$tool.txt
done
