# multi-segment staged hub kernels (TANGO_HUB_LANE=2): parity of all variants, Reddit layer A/B in one run
mkdir -p gpurun_out/r3b
timeout 1500 python -m pytest tests/test_gpu_layer.py -x -q > gpurun_out/r3b/tests.log 2>&1; echo rc=$? >> gpurun_out/r3b/tests.log
timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3b/base.json 2> gpurun_out/r3b/base.err
TANGO_HUB_LANE=2 timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3b/m2.json 2> gpurun_out/r3b/m2.err
timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3b/base2.json 2> gpurun_out/r3b/base2.err
TANGO_HUB_LANE=2 timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3b/m2b.json 2> gpurun_out/r3b/m2b.err
