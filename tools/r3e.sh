# 256-bit record stores in P1; P2 hub kernels multi-segment staged (TANGO_HUB_P2=2) vs staged: parity + A/B x2
mkdir -p gpurun_out/r3e
timeout 1800 python -m pytest tests/test_gpu_layer.py -x -q > gpurun_out/r3e/tests.log 2>&1; echo rc=$? >> gpurun_out/r3e/tests.log
for i in 1 2; do
timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3e/base$i.json 2> gpurun_out/r3e/base$i.err
TANGO_HUB_P2=2 timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3e/p2m$i.json 2> gpurun_out/r3e/p2m$i.err
done
