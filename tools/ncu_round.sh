#!/bin/bash
# ncu evidence for one config: launch list (one execute after warm-up) + full sets
cd "$(dirname "$0")/.."
C=${1:-c3}
python tools/profile_step.py $C 2 > gpurun_out/plain_$C.log 2>&1 || { cat gpurun_out/plain_$C.log; exit 1; }
# launches of the 3rd execute (skip plan-time and 2 warm-up executes: match only hot kernels)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'k_(split|col|row|crt|finish)' -s 16 -c 8 --csv --log-file gpurun_out/launches_$C.csv \
    python tools/profile_step.py $C 2 > gpurun_out/ncu_launch_$C.log 2>&1
for K in ${KERNELS:-k_row_fused k_col_inv k_crt_finish}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
      -o gpurun_out/prof_${C}_$K -f python tools/profile_step.py $C 2 > gpurun_out/ncu_full_${C}_$K.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
