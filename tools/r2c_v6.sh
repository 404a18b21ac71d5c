# v6 dataflow: layer parity on the GPU, then the Reddit-shaped layer bench
mkdir -p gpurun_out/r2c
timeout 900 python -m pytest tests/test_gpu_layer.py -x -q > gpurun_out/r2c/tests.log 2>&1; echo rc=$? >> gpurun_out/r2c/tests.log
timeout 900 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2c/bench_reddit.json 2> gpurun_out/r2c/bench_reddit.err
timeout 600 python bench.py --workload arxiv --steps 10 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2c/bench_arxiv.json 2> gpurun_out/r2c/bench_arxiv.err
