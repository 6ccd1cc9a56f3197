cd /root/repo; mkdir -p gpurun_out/mg
timeout 1500 python -m pytest tests/test_gpu_shard.py tests/test_gpu_parity.py tests/test_gpu_image.py -x -q > gpurun_out/mg/tests.log 2>&1; tail -2 gpurun_out/mg/tests.log
timeout 600 python bench.py --gpus 2 --backend gloo --one-device --config c2 --steps 5 --warmup 3 --no-cpu > gpurun_out/mg/c2_g2.json 2> gpurun_out/mg/c2_g2.err; tail -c 600 gpurun_out/mg/c2_g2.json; tail -3 gpurun_out/mg/c2_g2.err
timeout 600 python bench.py --gpus 3 --backend gloo --one-device --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/mg/c5_g3.json 2> gpurun_out/mg/c5_g3.err; python -c "import json;d=json.loads(open('gpurun_out/mg/c5_g3.json').read().splitlines()[-1]);print(d['n_gpus'],d['config']['global_batch'],d['bitwise_vs_n1'],d['value'])"; tail -3 gpurun_out/mg/c5_g3.err
timeout 600 python bench.py --mode single --config c3 --steps 10 > gpurun_out/mg/single.json 2> gpurun_out/mg/single.err; cat gpurun_out/mg/single.json; tail -3 gpurun_out/mg/single.err
timeout 600 python bench.py --config c3 --steps 10 --no-cpu --no-extra > gpurun_out/mg/c3.json 2> gpurun_out/mg/c3.err; python tools/show_bench.py gpurun_out/mg/c3.json | head -3
for B in 2 4 8; do OZ_BENCH_BATCH=$B true; done
