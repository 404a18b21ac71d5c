mkdir -p gpurun_out
for hb in 2 4 8; do
  TANGO_HUB_BLOCKS_PER_SM=$hb timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --layer-only > gpurun_out/hub_arxiv_$hb.json 2>/dev/null
done
for hb in 2 4 8; do
  TANGO_HUB_BLOCKS_PER_SM=$hb timeout 600 python bench.py --workload products --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/hub_products_$hb.json 2>/dev/null
done
