# validation of the F-stats load batching: layer parity (all variants) + Reddit layer
mkdir -p gpurun_out/r3h
timeout 1500 python -m pytest tests/test_gpu_layer.py -x -q > gpurun_out/r3h/tests.log 2>&1; echo rc=$? >> gpurun_out/r3h/tests.log
timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3h/reddit.json 2> gpurun_out/r3h/reddit.err
