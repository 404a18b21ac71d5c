mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_int4.py -x -q > gpurun_out/gpu_v.log 2>&1; echo rc=$? >> gpurun_out/gpu_v.log
timeout 500 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_v.json 2> gpurun_out/bench_v.err
