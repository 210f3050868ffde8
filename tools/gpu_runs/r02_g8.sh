# r02 call 8 (1 GPU): compute-sanitizer over every kernel (small stream-ordered cases)
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize/kernels_small.py > gpurun_out/g8_sanitize_$tool.log 2>&1; echo $tool=$?; tail -3 gpurun_out/g8_sanitize_$tool.log
done
