# session-3 baseline: default bench (Reddit headline), launch list, ncu --set full of the Reddit v6 kernels, GPU suite
mkdir -p gpurun_out/r2s
nvidia-smi > gpurun_out/r2s/nvsmi.txt 2>&1
( time timeout 1200 python bench.py > gpurun_out/r2s/bench.json 2> gpurun_out/r2s/bench.err ) 2> gpurun_out/r2s/bench_time.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s/launches_reddit.csv python bench.py --workload reddit --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2s/ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k2_|k_quantize|k_gemm" -c 16 -o /tmp/ncu_reddit python bench.py --workload reddit --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2s/ncu_reddit.log 2>&1
python tools/ncu_summary.py /tmp/ncu_reddit.ncu-rep > gpurun_out/r2s/ncu_reddit.summary.txt 2>&1
python tools/ncu_stalls.py /tmp/ncu_reddit.ncu-rep > gpurun_out/r2s/stalls.txt 2>&1
cp /tmp/ncu_reddit.ncu-rep gpurun_out/r2s/ 2>/dev/null
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2s/tests.log 2>&1; echo rc=$? >> gpurun_out/r2s/tests.log
