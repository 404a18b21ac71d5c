mkdir -p gpurun_out/r2h
timeout 900 python -m pytest tests/test_gpu_layer.py -x -q > gpurun_out/r2h/tests.log 2>&1; echo rc=$? >> gpurun_out/r2h/tests.log
timeout 900 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2h/bench_reddit.json 2> gpurun_out/r2h/bench_reddit.err
timeout 600 python bench.py --workload arxiv --steps 10 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2h/bench_arxiv.json 2> gpurun_out/r2h/bench_arxiv.err
