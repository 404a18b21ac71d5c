# P1 scatter of ∂α into in-CSR order (P2 reads it coalesced), gather-address / fold-counter micro-opts,
# quantize strided streaming path, vectorised incidence SPMM: parity, Reddit layer, ncu of the changed kernels
mkdir -p gpurun_out/r2u
timeout 900 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_layer.py -x -q > gpurun_out/r2u/tests.log 2>&1; echo rc=$? >> gpurun_out/r2u/tests.log
TANGO_P2_GATHER=1 timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2u/reddit_gather.json 2> gpurun_out/r2u/reddit_gather.err
timeout 1200 python bench.py --workload reddit --extras arxiv,products --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2u/reddit.json 2> gpurun_out/r2u/reddit.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k2_bdst|k2_bsrc|k2_fagg_seg|k_quantize" -c 10 -o /tmp/ncu_u python bench.py --workload reddit --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2u/ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu_u.ncu-rep > gpurun_out/r2u/ncu_summary.txt 2>&1
python tools/ncu_stalls.py /tmp/ncu_u.ncu-rep > gpurun_out/r2u/stalls.txt 2>&1
cp /tmp/ncu_u.ncu-rep gpurun_out/r2u/
