mkdir -p gpurun_out/r2n
for g in 32 64 128; do TANGO_L2_FETCH=$g timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2n/g$g.json 2> gpurun_out/r2n/g$g.err; done
