#!/bin/bash
# Evidence pass, part 1: bench (all configs, c3 with cpu_baseline + reference arm) and the ncu
# launch list.  Part 2 (KERNELS="..." tools/round_evidence.sh full): ncu --set full captures,
# at most two per call (gpurun brings back <= 64 MiB).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ev
if [ "$1" = "full" ]; then
  for K in ${KERNELS:-k_row_fused k_col_inv_crt}; do
    ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
        -o gpurun_out/ev/prof_c3_$K -f python tools/profile_step.py c3 2 > gpurun_out/ev/ncu_full_$K.log 2>&1
  done
  ls -la gpurun_out/ev
  exit 0
fi
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/ev/smi.txt
python bench.py > gpurun_out/ev/bench_c3.json 2> gpurun_out/ev/bench_c3.err
for c in c1 c2 c4 c5; do python bench.py --config $c --no-cpu > gpurun_out/ev/bench_$c.json 2> gpurun_out/ev/bench_$c.err; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev/ref_c3.json 2> gpurun_out/ev/ref_c3.err
python tools/profile_step.py c3 2 > gpurun_out/ev/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'k_(split|col|row|crt|finish)' -s 16 -c 8 --csv --log-file gpurun_out/ev/launches_c3.csv \
    python tools/profile_step.py c3 2 > gpurun_out/ev/ncu_launch.log 2>&1
ls gpurun_out/ev
