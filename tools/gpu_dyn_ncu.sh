#!/bin/bash
# ncu sections of the dot kernel: static partition vs dynamic chunks
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for V in '{"block":256,"unroll":4,"waves":2}' '{"block":256,"unroll":4,"waves":1,"chunk":8192}'; do
  timeout 600 ncu --section SpeedOfLight --section Occupancy --section WarpStateStats --section InstructionStats --section LaunchStats \
      --clock-control none -k regex:dot_k -s 2 -c 1 python tools/profile_kernels.py dot "$V" 2>&1 | \
      grep -E "Duration|DRAM Throughput|Achieved Occupancy|Registers Per|Grid Size|Executed Instructions  |Stall|Warp Cycles Per Issued|Issued Warp|Theoretical Occ" 
  echo "----"
done
