# end-of-round confirmation on the final tree: smoke, full GPU suite, default bench, launch list
mkdir -p gpurun_out/r3n
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3n/smoke.log 2>&1; echo rc=$? >> gpurun_out/r3n/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r3n/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r3n/gpu_tests.log
( time timeout 1800 python bench.py > gpurun_out/r3n/bench.json 2> gpurun_out/r3n/bench.err ) 2> gpurun_out/r3n/bench_time.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3n/launches_reddit.csv python bench.py --workload reddit --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3n/ncu_launch.log 2>&1
