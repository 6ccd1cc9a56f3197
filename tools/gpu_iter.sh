#!/bin/bash
# quick GPU iteration: parity subset + bench stage breakdown
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4
for c in ${CONFIGS:-c3}; do
  python bench.py --config $c --no-cpu --steps ${STEPS:-10} > gpurun_out/it_$c.json 2> gpurun_out/it_$c.err || tail -5 gpurun_out/it_$c.err
  python tools/show_bench.py gpurun_out/it_$c.json
done
