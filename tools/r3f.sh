# primitives: partial slots for multi-chunk rows only (batches of 256 rows), deeper incidence loads;
# tango_sddmm_q on the warp kernels; P1 evict-first streams: prims + layer parity, μ benches, Reddit layer
mkdir -p gpurun_out/r3f
timeout 1200 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_layer.py -x -q > gpurun_out/r3f/tests.log 2>&1; echo rc=$? >> gpurun_out/r3f/tests.log
timeout 1500 python bench.py --workload reddit --extras arxiv,sddmm --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3f/bench.json 2> gpurun_out/r3f/bench.err
