mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_paths.py \
      > gpurun_out/r2_sanitizer_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/r2_sanitizer_$tool.log
done
timeout 900 compute-sanitizer --tool initcheck --print-limit 50 python tools/sanitize_paths.py --no-exchange \
    > gpurun_out/r2_sanitizer_initcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2_sanitizer_initcheck.log
