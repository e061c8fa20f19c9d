#!/bin/bash
# One GPU session: tests, smoke, bench, ncu evidence.  Outputs -> gpurun_out/
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
python -m paper_0911_3456_b200._build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
if [ -n "${NCU}" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --quick --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dot_k -s 3 -c 1 -o gpurun_out/prof_dot -f python bench.py --steps 5 --warmup 3 --quick --no-cpu > gpurun_out/ncu_full.log 2>&1
fi
ls -la gpurun_out
