mkdir -p gpurun_out/r2p
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2p/tests.log 2>&1; echo rc=$? >> gpurun_out/r2p/tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2p/bench.json 2> gpurun_out/r2p/bench.err
