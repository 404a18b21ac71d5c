# new primitives (fast incidence SPMM, weighted SPMM with row scale / amax, quantize without amax slot) + L2
# fetch-granularity sweep on the Reddit layer (P2's random ∂α gather)
mkdir -p gpurun_out/r2t
timeout 900 python -m pytest tests/test_gpu_primitives.py -x -q > gpurun_out/r2t/prims.log 2>&1; echo rc=$? >> gpurun_out/r2t/prims.log
for g in 32 64; do TANGO_L2_FETCH=$g timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2t/g$g.json 2> gpurun_out/r2t/g$g.err; done
timeout 1200 python bench.py --workload reddit --extras arxiv,products --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2t/arxiv_inc.json 2> gpurun_out/r2t/arxiv_inc.err
