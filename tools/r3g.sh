# last validation of the committed tree: smoke, full GPU suite, default bench (Reddit headline + extras incl. products)
mkdir -p gpurun_out/r3g
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3g/smoke.log 2>&1; echo rc=$? >> gpurun_out/r3g/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r3g/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r3g/gpu_tests.log
( time timeout 1800 python bench.py > gpurun_out/r3g/bench.json 2> gpurun_out/r3g/bench.err ) 2> gpurun_out/r3g/bench_time.log
