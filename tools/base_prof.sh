#!/bin/bash
# Baseline: bench c3 stage breakdown + source-level ncu of the two NTT kernels (c3).
cd "$(dirname "$0")/.."; mkdir -p gpurun_out/base
python bench.py --config c3 --no-cpu --steps 10 > gpurun_out/base/bench_c3.json 2> gpurun_out/base/bench_c3.err
python tools/profile_step.py c3 1 > gpurun_out/base/plain.log 2>&1 || exit 1
for K in k_row_fused k_col_inv_crt; do
  ncu --set full --import-source on --clock-control none -k regex:$K -s 1 -c 1 -o /tmp/b_$K -f \
    python tools/profile_step.py c3 1 > gpurun_out/base/ncu_$K.log 2>&1
  ncu -i /tmp/b_$K.ncu-rep --page raw --csv > gpurun_out/base/raw_$K.csv 2>&1
  ncu -i /tmp/b_$K.ncu-rep --page source --csv --print-source sass > gpurun_out/base/src_$K.csv 2>&1
done
ls -la gpurun_out/base
