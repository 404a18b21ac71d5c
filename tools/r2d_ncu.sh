# ncu --set full of the v6 kernels on the Reddit-shaped layer (one launch each)
mkdir -p gpurun_out/r2d
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k2_" -c 6 -o gpurun_out/r2d/reddit_v6 python bench.py --workload reddit --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2d/ncu.log 2>&1
