mkdir -p gpurun_out
( time timeout 1500 python bench.py --workload products --steps 10 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/bench_products.json 2> gpurun_out/bench_products.err ) 2> gpurun_out/products_time.log
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/products_time.log
