#!/bin/bash
# Build libozfft variants in parallel: tools/build_variants.sh "tag1:-DFOO=1 -DBAR=2" "tag2:..."
# -> variants/libozfft_<tag>.so (host objects from the regular build are reused).
cd "$(dirname "$0")/.."
python -m paper_2603_29129_b200.build > /dev/null || exit 1
B=paper_2603_29129_b200/_build
mkdir -p variants
for spec in "$@"; do
  tag=${spec%%:*}; flags=${spec#*:}
  ( /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
      $flags -Xcompiler -fPIC -c paper_2603_29129_b200/csrc/kernels.cu -o /tmp/k_$tag.o && \
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/libozfft_$tag.so \
      /tmp/k_$tag.o $B/capi.cpp.o $B/plan_host.cpp.o $B/version.cpp.o -lquadmath -cudart static && \
    echo "built $tag: $(cuobjdump -res-usage variants/libozfft_$tag.so | grep -A1 'k_row_fusedILi11ELb1E' | grep -o 'REG:[0-9]*')" ) &
done
wait
