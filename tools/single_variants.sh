#!/bin/bash
# single-transform shard path at N = 1 for the main build and variants/libozfft_<tag>.so
cd "$(dirname "$0")/.."
cp paper_2603_29129_b200/libozfft.so /tmp/libozfft_main.so
for tag in main "$@"; do
  [ "$tag" = main ] && f=/tmp/libozfft_main.so || f=variants/libozfft_$tag.so
  cp $f paper_2603_29129_b200/libozfft.so
  echo "== $tag"; python tools/single_prof.py c3 | grep -E "shard|crt_finish" | head -2
done
cp /tmp/libozfft_main.so paper_2603_29129_b200/libozfft.so
