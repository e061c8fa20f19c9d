#!/bin/bash
# C3 with the prelude's lean sin: bench's elementwise group (tuned + confirmed
# like the driver's run) and an ncu capture of the prefetch variant.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py --only elementwise --no-cpu > gpurun_out/c3_bench.json 2> gpurun_out/c3_bench.err
echo bench_rc=$?
PS_PREF='{"block":128,"unroll":1,"waves":4,"prefetch":true}'
timeout 600 ncu --set full --clock-control none --import-source on -k regex:polysin -s 2 -c 1 \
    -o gpurun_out/r2b_prof_polysin_pref -f python tools/profile_kernels.py polysin "$PS_PREF" > gpurun_out/r2b_prof_polysin_pref.log 2>&1
echo ncu_rc=$?
