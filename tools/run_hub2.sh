mkdir -p gpurun_out
for hb in 1 2 1 2; do
  TANGO_HUB_BLOCKS_PER_SM=$hb timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --layer-only 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$hb', round(d['value'],4))" >> gpurun_out/hub2.log
done
