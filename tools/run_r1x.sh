mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_partitioned.py -x -q > gpurun_out/gpu_x.log 2>&1; echo rc=$? >> gpurun_out/gpu_x.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train-step --nccl-single > gpurun_out/bench_x.json 2> gpurun_out/bench_x.err; echo rc=$? >> gpurun_out/gpu_x.log
