# batched work-queue claims: GAT parity (sparse + dense + variants) and partitioned / model suites, Reddit + arxiv layers
mkdir -p gpurun_out/r3j
timeout 1800 python -m pytest tests/test_gpu_layer.py tests/test_gpu_partitioned.py tests/test_gpu_model.py -x -q > gpurun_out/r3j/tests.log 2>&1; echo rc=$? >> gpurun_out/r3j/tests.log
for i in 1 2; do
timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3j/reddit$i.json 2> gpurun_out/r3j/reddit$i.err
done
timeout 600 python bench.py --workload arxiv --steps 10 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3j/arxiv.json 2> gpurun_out/r3j/arxiv.err
