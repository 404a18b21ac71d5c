# P3 reads P1's out-CSR signed α (al_out) instead of recomputing α: parity (all variants), Reddit layer x2
mkdir -p gpurun_out/r3d
timeout 1800 python -m pytest tests/test_gpu_layer.py -x -q > gpurun_out/r3d/tests.log 2>&1; echo rc=$? >> gpurun_out/r3d/tests.log
for i in 1 2; do
timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3d/rec$i.json 2> gpurun_out/r3d/rec$i.err
done
