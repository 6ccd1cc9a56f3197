cd /root/repo
cp paper_2603_29129_b200/libozfft.so /tmp/orig.so
for v in s1 s2; do cp variants/libozfft_$v.so paper_2603_29129_b200/libozfft.so
 for mode in "--accum image" "--accum image --conv cyclic"; do
  python bench.py $mode --no-cpu --no-extra --steps 10 > gpurun_out/v.json 2>/dev/null; echo "== $v $mode"; python tools/show_bench.py gpurun_out/v.json | grep "GF/s  \|col_inv"; done; done
cp /tmp/orig.so paper_2603_29129_b200/libozfft.so
