#!/bin/bash
# Bench several prebuilt libozfft variants (variants/libozfft_<tag>.so) on the same box.
cd "$(dirname "$0")/.."
cp paper_2603_29129_b200/libozfft.so /tmp/libozfft_orig.so
for f in variants/libozfft_*.so; do
  tag=$(basename $f .so | sed 's/libozfft_//')
  cp $f paper_2603_29129_b200/libozfft.so
  python bench.py --config ${CONFIG:-c3} --no-cpu --steps 10 > gpurun_out/var_${CONFIG:-c3}_$tag.json 2>/dev/null
  echo "== $tag"; python tools/show_bench.py gpurun_out/var_${CONFIG:-c3}_$tag.json 2>/dev/null | grep -E "GF/s|${SHOW:-row_fused|col_inv}"
done
cp /tmp/libozfft_orig.so paper_2603_29129_b200/libozfft.so
