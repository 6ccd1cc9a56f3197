#!/bin/bash
# ncu --set full of the given kernels (c3, tools/profile_step.py), exported on the box as CSV
# pages (details, raw, source) so that gpurun_out stays small; summarise here with
#   python tools/summarize_ncu.py gpurun_out/ev <tag>
cd "$(dirname "$0")/.."; mkdir -p gpurun_out/ev
python tools/profile_step.py c3 2 > gpurun_out/ev/plain_full.log 2>&1 || exit 1
for K in ${KERNELS:-k_row_fused k_col_inv_crt}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
      -o /tmp/prof_c3_$K -f python tools/profile_step.py c3 2 > gpurun_out/ev/ncu_full_$K.log 2>&1
  for pg in details raw; do ncu -i /tmp/prof_c3_$K.ncu-rep --page $pg --csv > gpurun_out/ev/prof_c3_${K}_$pg.csv; done
  ncu -i /tmp/prof_c3_$K.ncu-rep --page source --csv --print-source sass > gpurun_out/ev/prof_c3_${K}_sass.csv
done
ls -la gpurun_out/ev
