# software-pipelined lane-parallel hub kernels, P1 deferred dot correction + lazy record unpack: v6 parity, Reddit layer
mkdir -p gpurun_out/r2w
timeout 900 python -m pytest tests/test_gpu_layer.py -x -q > gpurun_out/r2w/tests.log 2>&1; echo rc=$? >> gpurun_out/r2w/tests.log
timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2w/reddit.json 2> gpurun_out/r2w/reddit.err
TANGO_P2_GATHER=1 timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2w/reddit_gather.json 2> gpurun_out/r2w/reddit_gather.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"_hub|k2_bsrc1_seg" -c 6 -o /tmp/ncu_w python bench.py --workload reddit --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2w/ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu_w.ncu-rep > gpurun_out/r2w/ncu_summary.txt 2>&1
python tools/ncu_stalls.py /tmp/ncu_w.ncu-rep > gpurun_out/r2w/stalls.txt 2>&1
cp /tmp/ncu_w.ncu-rep gpurun_out/r2w/
