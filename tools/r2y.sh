# defaults back to gather + staged hubs, IMAD.HI reverted: layer parity (incl. the env variants), default bench,
# the multi-head SPMM sweep through the standalone primitive (arxiv extras)
mkdir -p gpurun_out/r2y
timeout 1200 python -m pytest tests/test_gpu_layer.py tests/test_gpu_primitives.py -x -q > gpurun_out/r2y/tests.log 2>&1; echo rc=$? >> gpurun_out/r2y/tests.log
( time timeout 1200 python bench.py > gpurun_out/r2y/bench.json 2> gpurun_out/r2y/bench.err ) 2> gpurun_out/r2y/bench_time.log
timeout 900 python bench.py --workload reddit --extras arxiv,sddmm --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2y/arxiv_sddmm.json 2> gpurun_out/r2y/arxiv_sddmm.err
