mkdir -p gpurun_out
( time timeout 1500 python bench.py --workload reddit --steps 10 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/bench_reddit.json 2> gpurun_out/bench_reddit.err ) 2> gpurun_out/reddit_time.log
