mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_int4.py -x -q > gpurun_out/gpu_w.log 2>&1; echo rc=$? >> gpurun_out/gpu_w.log
timeout 500 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_w.json 2> gpurun_out/bench_w.err
timeout 600 ncu --set full --clock-control none -k regex:k_sddmm_dot_e -c 2 -o gpurun_out/dot_r1w python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_dot.log 2>&1
