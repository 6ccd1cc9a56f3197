#!/bin/bash
# A/B of prebuilt libozfft variants on one box: the -m gpu suite against the in-tree build,
# then VARIANTS (default: every variants/libozfft_*.so) benched REPS times in turn on CONFIGS.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ab
[ -n "$NOTEST" ] || timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
cp paper_2603_29129_b200/libozfft.so /tmp/cur.so
VARIANTS=${VARIANTS:-$(ls variants/libozfft_*.so | sed 's/.*libozfft_//; s/\.so//')}
for rep in $(seq 1 ${REPS:-2}); do for v in $VARIANTS; do
  cp variants/libozfft_$v.so paper_2603_29129_b200/libozfft.so
  for c in ${CONFIGS:-c3 c2}; do python bench.py --config $c --no-cpu --steps 20 > gpurun_out/ab/${v}_${c}_$rep.json 2>/dev/null; done
done; done
cp /tmp/cur.so paper_2603_29129_b200/libozfft.so
for f in gpurun_out/ab/*.json; do python tools/show_bench.py $f 2>/dev/null | grep -E "GF/s|row_fused" | head -2 | tr '\n' ' '; echo; done
