#!/bin/bash
# A/B on one box: parity subset on the in-tree build, then bench stage lines per variant.
#   TESTS="tests/test_gpu_parity.py" CONFIGS="c3" tools/ab.sh tag1 tag2 ...
cd "$(dirname "$0")/.."; mkdir -p gpurun_out/ab
if [ -n "${TESTS-tests/test_gpu_parity.py}" ]; then
  timeout 900 python -m pytest ${TESTS-tests/test_gpu_parity.py} -x -q > gpurun_out/ab/tests.log 2>&1
  tail -3 gpurun_out/ab/tests.log
fi
cp paper_2603_29129_b200/libozfft.so /tmp/libozfft_main.so
for vt in $VTEST; do  # parity of variant builds too
  cp variants/libozfft_$vt.so paper_2603_29129_b200/libozfft.so
  timeout 900 python -m pytest ${VTESTS:-tests/test_gpu_parity.py tests/test_gpu_configs.py} -x -q > gpurun_out/ab/tests_$vt.log 2>&1
  echo "tests $vt: $(tail -1 gpurun_out/ab/tests_$vt.log)"
done
cp /tmp/libozfft_main.so paper_2603_29129_b200/libozfft.so
for tag in main "$@"; do
  [ "$tag" = main ] && f=/tmp/libozfft_main.so || f=variants/libozfft_$tag.so
  cp $f paper_2603_29129_b200/libozfft.so
  for c in ${CONFIGS:-c3}; do
    python bench.py --config $c --no-cpu --steps ${STEPS:-10} > gpurun_out/ab/${tag}_$c.json 2> gpurun_out/ab/${tag}_$c.err
    echo "== $tag $c"; python tools/show_bench.py gpurun_out/ab/${tag}_$c.json 2>&1 | grep -E "GF/s|${SHOW:-row_fused|col_inv}" | head -4
  done
done
cp /tmp/libozfft_main.so paper_2603_29129_b200/libozfft.so
