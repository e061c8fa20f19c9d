#!/bin/bash
# Round-2 ncu evidence (run under gpurun from the repo root).  One GPU.
set -u
mkdir -p gpurun_out
DOT='{"block":256,"unroll":1,"waves":2}'
PS_RING='{"block":512,"unroll":2,"waves":2,"stages":2}'
PS_PREF='{"block":256,"unroll":1,"waves":1,"prefetch":true}'
AXPY='{"block":128,"unroll":1,"waves":0}'
# 1. full captures of the top kernels (variants the bench picks)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dot_k -s 2 -c 1 \
    -o gpurun_out/r2_prof_dot -f python tools/profile_kernels.py dot "$DOT" > gpurun_out/r2_prof_dot.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:polysin -s 2 -c 1 \
    -o gpurun_out/r2_prof_polysin_ring -f python tools/profile_kernels.py polysin "$PS_RING" > gpurun_out/r2_prof_polysin_ring.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:polysin -s 2 -c 1 \
    -o gpurun_out/r2_prof_polysin_pref -f python tools/profile_kernels.py polysin "$PS_PREF" > gpurun_out/r2_prof_polysin_pref.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:axpy -s 2 -c 1 \
    -o gpurun_out/r2_prof_axpy -f python tools/profile_kernels.py axpy "$AXPY" > gpurun_out/r2_prof_axpy.log 2>&1
# 2. launch list of the bench command (headline only; tuning launches included)
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 6000 --csv --log-file gpurun_out/r2_launches_bench.csv \
    python bench.py --quick --no-cpu --steps 20 --warmup 5 > gpurun_out/r2_launches_bench.json 2> gpurun_out/r2_launches_bench.err
echo done
