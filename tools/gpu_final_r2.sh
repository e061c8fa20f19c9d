#!/bin/bash
# End-of-round validation on one B200 (outputs -> gpurun_out/final_*):
# smoke, the GPU suite, the driver-style bench (N = 1), the reference arm,
# --gpus 2 with both ranks on this GPU, the bench command's ncu launch list
# and one ncu --set full capture of the headline kernel.
set -u
mkdir -p gpurun_out
nvidia-smi > gpurun_out/final_nvidia_smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/final_pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err; echo "bench rc=$?" >> gpurun_out/final_bench_n1.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final_bench_reference.json 2> gpurun_out/final_bench_reference.err
timeout 1200 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/final_bench_g2.json 2> gpurun_out/final_bench_g2.err; echo "g2 rc=$?" >> gpurun_out/final_bench_g2.err
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 6000 --csv --log-file gpurun_out/final_launches_bench.csv \
    python bench.py --quick --no-cpu --steps 20 --warmup 5 > gpurun_out/final_launches_bench.json 2> gpurun_out/final_launches_bench.err
DOT=$(python -c "import json; d=json.loads(open('gpurun_out/final_bench_n1.json').read().strip().splitlines()[-1])['config']; print(json.dumps({k[8:]: d[k] for k in ('variant_block','variant_unroll','variant_waves')}))" 2>/dev/null || echo '{"block":512,"unroll":1,"waves":2}')
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dot_k -s 2 -c 1 \
    -o gpurun_out/final_prof_dot -f python tools/profile_kernels.py dot "$DOT" > gpurun_out/final_prof_dot.log 2>&1
echo done
