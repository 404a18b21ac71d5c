mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_layer.py tests/test_gpu_model.py -x -q > gpurun_out/gemmfix.log 2>&1; echo rc=$? >> gpurun_out/gemmfix.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --layer-only 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('arxiv', round(d['value'],4), d['kernel_roofline']['gemm_store'])" >> gpurun_out/gemmfix.log
timeout 1500 python bench.py --workload reddit --steps 10 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/bench_reddit3.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_reddit3.json')); print('reddit', round(d['value'],3), d['kernel_roofline']['gemm_store'])" >> gpurun_out/gemmfix.log
