# GEMM fp32 epilogue with float2 stores: GEMM / layer / model parity, Reddit layer (gemm_store time), arxiv layer
mkdir -p gpurun_out/r3m
timeout 1500 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_layer.py tests/test_gpu_model.py -x -q > gpurun_out/r3m/tests.log 2>&1; echo rc=$? >> gpurun_out/r3m/tests.log
timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3m/reddit.json 2> gpurun_out/r3m/reddit.err
timeout 600 python bench.py --workload arxiv --steps 10 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3m/arxiv.json 2> gpurun_out/r3m/arxiv.err
