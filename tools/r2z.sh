# standalone primitives on row blocks (no CSR search), weighted SPMM with 16-column lanes, int8-α SPMM:
# parity + the μ benchmarks (incidence SPMM on arxiv / products, multi-head SPMM sweep incl. int8-α)
mkdir -p gpurun_out/r2z
timeout 900 python -m pytest tests/test_gpu_primitives.py -x -q > gpurun_out/r2z/tests.log 2>&1; echo rc=$? >> gpurun_out/r2z/tests.log
timeout 1500 python bench.py --workload reddit --extras arxiv,products,sddmm --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2z/bench.json 2> gpurun_out/r2z/bench.err
