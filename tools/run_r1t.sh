mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_model.py -x -q > gpurun_out/gpu_t.log 2>&1; echo rc=$? >> gpurun_out/gpu_t.log
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err
