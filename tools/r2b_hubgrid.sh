# hub-grid occupancy experiment on the Reddit-shaped layer (existing kernels)
mkdir -p gpurun_out/r2b
for hb in 3 6; do
  TANGO_HUB_BLOCKS_PER_SM=$hb timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2b/bench_hb$hb.json 2> gpurun_out/r2b/bench_hb$hb.err
done
