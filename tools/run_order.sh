mkdir -p gpurun_out
for o in random degree; do
  timeout 1200 python bench.py --workload products --order $o --steps 5 --warmup 3 --no-cpu-baseline --layer-only 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o', round(d['value'],3), d['kernel_roofline'])" >> gpurun_out/order.log
  timeout 600 python bench.py --workload arxiv --order $o --steps 20 --warmup 3 --no-cpu-baseline --layer-only 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('arxiv $o', round(d['value'],4))" >> gpurun_out/order.log
done
