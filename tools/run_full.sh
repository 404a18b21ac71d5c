mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_full.log 2>&1; echo rc=$? >> gpurun_out/gpu_full.log
