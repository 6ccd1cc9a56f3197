#!/bin/bash
# Source-level ncu of the three c1 kernels (exported as CSV on the box)
cd "$(dirname "$0")/.."; mkdir -p gpurun_out/c1
python tools/profile_step.py c1 2 > gpurun_out/c1/plain.log 2>&1 || exit 1
for K in k_split_cluster k_row_fused k_crt_finish; do
  ncu --set full --import-source on --clock-control none -k regex:$K -s 2 -c 1 -o /tmp/c1_$K -f \
    python tools/profile_step.py c1 2 > gpurun_out/c1/ncu_$K.log 2>&1
  ncu -i /tmp/c1_$K.ncu-rep --page raw --csv > gpurun_out/c1/raw_$K.csv 2>&1
  ncu -i /tmp/c1_$K.ncu-rep --page source --csv --print-source sass > gpurun_out/c1/src_$K.csv 2>&1
done
