cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_small.py tests/test_gpu_configs.py tests/test_gpu_fault.py -x -q 2>&1 | tail -2
cp paper_2603_29129_b200/libozfft.so /tmp/cur.so
for rep in 1 2; do for v in base canon0; do
  cp variants/libozfft_$v.so paper_2603_29129_b200/libozfft.so
  for c in c3 c2; do python bench.py --config $c --no-cpu --steps 20 > gpurun_out/ab/${v}_${c}_$rep.json 2>/dev/null; done
done; done
cp /tmp/cur.so paper_2603_29129_b200/libozfft.so
for f in gpurun_out/ab/*.json; do python tools/show_bench.py $f | head -1; python tools/show_bench.py $f | grep row_fused; done
