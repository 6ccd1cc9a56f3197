#!/bin/bash
# Kernel durations (ncu gpu__time_duration, cold cache, serialised) of one forward execute
# per config for the main build and each variants/libozfft_<tag>.so:
#   tools/kernel_times.sh "c1 c2 c3" [kernel-regex]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFGS=${1:-"c1 c2 c3"}
KRE=${2:-.}
cp paper_2603_29129_b200/libozfft.so /tmp/libozfft_main.so
for f in /tmp/libozfft_main.so variants/libozfft_*.so; do
  tag=$(basename $f .so | sed 's/libozfft_//')
  cp $f paper_2603_29129_b200/libozfft.so
  for c in $CFGS; do
    ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:$KRE" --csv \
      --log-file gpurun_out/kt_${tag}_$c.csv python tools/profile_step.py $c 1 > /dev/null 2>&1
  done
done
cp /tmp/libozfft_main.so paper_2603_29129_b200/libozfft.so
