#!/bin/bash
# ncu --set full of the c3 split kernels (main build and variants/libozfft_ept4.so); raw
# metric pages as CSV (the reports themselves stay on the box).
cd "$(dirname "$0")/.."; mkdir -p gpurun_out
cp paper_2603_29129_b200/libozfft.so /tmp/main.so
for v in main ${VARIANTS}; do
  [ $v != main ] && cp variants/libozfft_$v.so paper_2603_29129_b200/libozfft.so
  ncu --set full --clock-control none -k regex:k_split_max -s 5 -c 1 -o /tmp/split_max_$v -f python tools/profile_step.py c3 1 > /dev/null 2>&1
  ncu --set full --clock-control none -k regex:k_split_digits -s 1 -c 1 -o /tmp/split_dig_$v -f python tools/profile_step.py c3 1 > /dev/null 2>&1
  for k in split_max split_dig; do
    ncu -i /tmp/${k}_$v.ncu-rep --page raw --csv > gpurun_out/raw_${k}_$v.csv 2>&1
    ncu -i /tmp/${k}_$v.ncu-rep --page details --csv > gpurun_out/det_${k}_$v.csv 2>&1
  done
done
cp /tmp/main.so paper_2603_29129_b200/libozfft.so
