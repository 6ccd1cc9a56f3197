#!/bin/bash
# Iteration: GPU tests ($TESTS), bench c3 stages, source-level ncu of $KERNEL (c3).
cd "$(dirname "$0")/.."; mkdir -p gpurun_out/it
timeout 1200 python -m pytest ${TESTS:-tests/test_gpu_parity.py} -x -q > gpurun_out/it/tests.log 2>&1; tail -3 gpurun_out/it/tests.log
for c in ${CONFIGS:-c3}; do
python bench.py --config $c --no-cpu --steps 10 > gpurun_out/it/bench_$c.json 2> gpurun_out/it/bench_$c.err
python tools/show_bench.py gpurun_out/it/bench_$c.json | head -8
done
if [ -n "$KERNEL" ]; then
python tools/profile_step.py c3 1 > gpurun_out/it/plain.log 2>&1 || exit 1
for K in $KERNEL; do
ncu --set full --import-source on --clock-control none -k regex:$K -s 1 -c 1 -o /tmp/it_$K -f \
  python tools/profile_step.py c3 1 > gpurun_out/it/ncu_$K.log 2>&1
ncu -i /tmp/it_$K.ncu-rep --page raw --csv > gpurun_out/it/raw_$K.csv 2>&1
ncu -i /tmp/it_$K.ncu-rep --page source --csv --print-source sass > gpurun_out/it/src_$K.csv 2>&1
done
fi
