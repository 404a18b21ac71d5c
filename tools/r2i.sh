mkdir -p gpurun_out/r2i
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2i/tests.log 2>&1; echo rc=$? >> gpurun_out/r2i/tests.log
timeout 900 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2i/bench_reddit.json 2> gpurun_out/r2i/bench_reddit.err
