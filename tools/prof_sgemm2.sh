mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sgemm2 -c 3 -o gpurun_out/sgemm_r1zz python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_sg2.log 2>&1
