cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/sm
timeout 600 python -m pytest tests/test_gpu_small.py tests/test_gpu_fault.py -x -q 2>&1 | tail -3
for z in 4 2 1; do OZFFT_SMALL_Z=$z python bench.py --config c1 --no-cpu > gpurun_out/sm/c1_z$z.json 2>/dev/null; python tools/show_bench.py gpurun_out/sm/c1_z$z.json | head -2; done
OZFFT_SMALL_FUSED=0 python bench.py --config c1 --no-cpu > gpurun_out/sm/c1_old.json 2>/dev/null; python tools/show_bench.py gpurun_out/sm/c1_old.json | head -1
cp variants/libozfft_smt.so paper_2603_29129_b200/libozfft.so
for z in 4 2; do OZFFT_SMALL_Z=$z python tools/small_phases.py 1024 20; done
