#!/bin/bash
# Bench prebuilt variants (variants/libozfft_<tag>.so) in several plan modes:
#   MODES="--conv cyclic|--accum image" VARIANTS="a b" SHOW=col_inv tools/variant_modes.sh
cd "$(dirname "$0")/.."
cp paper_2603_29129_b200/libozfft.so /tmp/orig.so
IFS='|' read -ra MS <<< "${MODES:- }"
for v in ${VARIANTS:-$(ls variants | sed 's/libozfft_//;s/.so//')}; do
  cp variants/libozfft_$v.so paper_2603_29129_b200/libozfft.so
  for mode in "${MS[@]}"; do
    python bench.py $mode --config ${CONFIG:-c3} --no-cpu --no-extra --steps 10 > gpurun_out/v.json 2>/dev/null
    echo "== $v [$mode]"; python tools/show_bench.py gpurun_out/v.json | grep "GF/s  \|${SHOW:-col_inv}"
  done
done
cp /tmp/orig.so paper_2603_29129_b200/libozfft.so
