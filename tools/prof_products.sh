mkdir -p gpurun_out
timeout 1700 ncu --set full --clock-control none -k regex:"k_fwd_agg4|k_bwd_src4" -c 4 -o gpurun_out/products_r1y python bench.py --workload products --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/ncu_products.log 2>&1
