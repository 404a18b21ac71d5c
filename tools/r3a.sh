# α stored by F-agg for P2: layer parity (incl. the env variants), Reddit layer, launch list
mkdir -p gpurun_out/r3a
timeout 1500 python -m pytest tests/test_gpu_layer.py -x -q > gpurun_out/r3a/tests.log 2>&1; echo rc=$? >> gpurun_out/r3a/tests.log
timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3a/reddit.json 2> gpurun_out/r3a/reddit.err
TANGO_ALPHA_RECOMPUTE=1 timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3a/reddit_recompute.json 2> gpurun_out/r3a/reddit_recompute.err
