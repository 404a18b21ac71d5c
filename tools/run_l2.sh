mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --layer-only 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],4), d['kernel_ms_per_step']['quantize'], d['kernel_ms_per_step']['absmax'])" >> gpurun_out/l2.log
done
timeout 300 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_layer.py -x -q 2>&1 | tail -1 >> gpurun_out/l2.log
