# lane-parallel hub segments (F-stats Σ, P2a, P2b, P3) + dense v6 parity cases + argument validation:
# full GPU suite, Reddit layer (lane vs staged hubs), launch list, ncu of the new kernels
mkdir -p gpurun_out/r2v
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2v/tests.log 2>&1; echo rc=$? >> gpurun_out/r2v/tests.log
TANGO_P2_GATHER=1 timeout 600 python -m pytest tests/test_gpu_layer.py -x -q -k v6 > gpurun_out/r2v/tests_gather.log 2>&1; echo rc=$? >> gpurun_out/r2v/tests_gather.log
TANGO_HUB_STAGED=1 timeout 600 python -m pytest tests/test_gpu_layer.py -x -q -k v6 > gpurun_out/r2v/tests_staged.log 2>&1; echo rc=$? >> gpurun_out/r2v/tests_staged.log
timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2v/reddit.json 2> gpurun_out/r2v/reddit.err
TANGO_HUB_STAGED=1 timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2v/reddit_staged.json 2> gpurun_out/r2v/reddit_staged.err
TANGO_P2_GATHER=1 timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2v/reddit_gather.json 2> gpurun_out/r2v/reddit_gather.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2v/launches_reddit.csv python bench.py --workload reddit --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2v/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"_hub|k2_fagg_seg|k2_bsrc1_seg" -c 8 -o /tmp/ncu_v python bench.py --workload reddit --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2v/ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu_v.ncu-rep > gpurun_out/r2v/ncu_summary.txt 2>&1
python tools/ncu_stalls.py /tmp/ncu_v.ncu-rep > gpurun_out/r2v/stalls.txt 2>&1
cp /tmp/ncu_v.ncu-rep gpurun_out/r2v/
