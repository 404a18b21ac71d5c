set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_layer.py tests/test_gpu_bits.py -x -q > gpurun_out/gpu_q.log 2>&1; echo rc=$? >> gpurun_out/gpu_q.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1r.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-train-step > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_quantize -s 6 -c 6 -o gpurun_out/quant_r1r python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-train-step > gpurun_out/ncu_q.log 2>&1
ls -la gpurun_out
