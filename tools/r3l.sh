# P3 hub segments multi-segment staged with P1's out-CSR α (TANGO_HUB_P3=2) vs staged: parity + A/B x2
mkdir -p gpurun_out/r3l
timeout 1500 python -m pytest tests/test_gpu_layer.py -x -q > gpurun_out/r3l/tests.log 2>&1; echo rc=$? >> gpurun_out/r3l/tests.log
for i in 1 2; do
timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3l/base$i.json 2> gpurun_out/r3l/base$i.err
TANGO_HUB_P3=2 timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3l/p3m$i.json 2> gpurun_out/r3l/p3m$i.err
done
