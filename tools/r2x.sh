# dataflow variants on the Reddit layer (IMAD.HI top-byte conversion, FS1 on int8 codes, hub ‖ tile streams):
# A gather+staged, B scatter+lane, C gather+lane; v6 parity under A and B
mkdir -p gpurun_out/r2x
TANGO_P2_GATHER=1 TANGO_HUB_STAGED=1 timeout 600 python -m pytest tests/test_gpu_layer.py -x -q > gpurun_out/r2x/tests_A.log 2>&1; echo rc=$? >> gpurun_out/r2x/tests_A.log
timeout 600 python -m pytest tests/test_gpu_layer.py -x -q > gpurun_out/r2x/tests_B.log 2>&1; echo rc=$? >> gpurun_out/r2x/tests_B.log
TANGO_P2_GATHER=1 TANGO_HUB_STAGED=1 timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2x/A.json 2> gpurun_out/r2x/A.err
timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2x/B.json 2> gpurun_out/r2x/B.err
TANGO_P2_GATHER=1 timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2x/C.json 2> gpurun_out/r2x/C.err
