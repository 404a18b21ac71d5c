mkdir -p gpurun_out/r2k
timeout 600 compute-sanitizer --tool memcheck --show-backtrace device python -m pytest tests/test_gpu_layer.py -x -q -k "ragged and not recompute" > gpurun_out/r2k/memcheck.log 2>&1
tail -60 gpurun_out/r2k/memcheck.log > gpurun_out/r2k/memcheck_tail.log
