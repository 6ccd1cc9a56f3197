#!/bin/bash
# Source-level ncu of k_small_fused at c1 (exported as CSV on the box)
cd "$(dirname "$0")/.."; mkdir -p gpurun_out/c1
python tools/profile_step.py c1 2 > gpurun_out/c1/plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_small_fused -s 2 -c 1 \
    --warp-sampling-interval 0 -o /tmp/c1_small -f python tools/profile_step.py c1 2 > gpurun_out/c1/ncu_small.log 2>&1
ncu -i /tmp/c1_small.ncu-rep --page raw --csv > gpurun_out/c1/raw_small.csv 2>&1
ncu -i /tmp/c1_small.ncu-rep --page source --csv --print-source sass > gpurun_out/c1/src_small.csv 2>&1
ncu -i /tmp/c1_small.ncu-rep --page source --csv --print-source cuda > gpurun_out/c1/srccu_small.csv 2>&1
ls -la gpurun_out/c1
