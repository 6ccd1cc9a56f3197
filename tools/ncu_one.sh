#!/bin/bash
# ncu --set full of one kernel (regex $1) in config $2 (launch skip $3, default 1); writes
# the raw metric page and the source-level SASS page (CSV) to gpurun_out/<tag>_*.csv.
cd "$(dirname "$0")/.."; mkdir -p gpurun_out
tag=${4:-$1_$2}
ncu --set full --import-source on --clock-control none -k regex:$1 -s ${3:-1} -c 1 -o /tmp/one_$tag -f \
  python tools/profile_step.py $2 1 > /dev/null 2>&1
ncu -i /tmp/one_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv 2>&1
ncu -i /tmp/one_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$tag.csv 2>&1
