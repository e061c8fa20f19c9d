#!/bin/bash
# compute-sanitizer over every template path (tools/sanitize_paths.py), plus
# ncu captures of the C4 reduction kernels with the bench's variants.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_paths.py \
      > gpurun_out/r2_sanitizer_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/r2_sanitizer_$tool.log
done
timeout 900 compute-sanitizer --tool initcheck --print-limit 50 python tools/sanitize_paths.py --no-exchange \
    > gpurun_out/r2_sanitizer_initcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2_sanitizer_initcheck.log
for k in maxabs sumsq sum_i64; do
  case $k in maxabs) V='{"block":1024,"unroll":1,"waves":2}';; sumsq) V='{"block":256,"unroll":1,"waves":2}';; sum_i64) V='{"block":256,"unroll":8,"waves":2}';; esac
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$([ $k = sum_i64 ] && echo sum_k || echo $k) -s 2 -c 1 \
      -o gpurun_out/r2_prof_$k -f python tools/profile_kernels.py $k "$V" > gpurun_out/r2_prof_$k.log 2>&1
done
