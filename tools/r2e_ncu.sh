mkdir -p gpurun_out/r2e
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k2_fagg|k2_bsrc1" -c 2 -o gpurun_out/r2e/reddit_g7 python bench.py --workload reddit --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2e/ncu.log 2>&1
