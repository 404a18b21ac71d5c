mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_layer.py tests/test_gpu_model.py tests/test_gpu_partitioned.py -x -q > gpurun_out/gpu_s.log 2>&1; echo rc=$? >> gpurun_out/gpu_s.log
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_quantize -s 10 -c 1 -o gpurun_out/quant_r1s python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-train-step > gpurun_out/ncu_q.log 2>&1
