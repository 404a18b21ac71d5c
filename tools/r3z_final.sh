# round-2 final evidence: ncu of one Reddit layer step first (its DRAM / L2 bytes feed the bench's roofline
# through profiles/ncu_traffic.json), then the default bench, smoke, the full GPU suite, the reference arm,
# the launch list and compute-sanitizer memcheck of the new code
mkdir -p gpurun_out/final
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"k2_|k_quantize|k_gemm" -c 24 -o /tmp/ncu_final python bench.py --workload reddit --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/final/ncu_full.log 2>&1
python tools/ncu_to_traffic.py /tmp/ncu_final.ncu-rep reddit r3_final_reddit > gpurun_out/final/traffic.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/final/ncu_traffic.json
python tools/ncu_summary.py /tmp/ncu_final.ncu-rep > gpurun_out/final/ncu_summary.txt 2>&1
python tools/ncu_stalls.py /tmp/ncu_final.ncu-rep > gpurun_out/final/ncu_stalls.txt 2>&1
ls -la /tmp/ncu_final.ncu-rep > gpurun_out/final/ncu_rep_size.txt   # the report stays on the box (64 MiB return limit)
python tools/ncu_hot.py /tmp/ncu_final.ncu-rep k2_bsrc1_seg > gpurun_out/final/hot_bsrc1_seg.txt 2>&1
python tools/ncu_hot.py /tmp/ncu_final.ncu-rep k2_fagg_seg > gpurun_out/final/hot_fagg_seg.txt 2>&1
( time timeout 1500 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err ) 2> gpurun_out/final/bench_time.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo rc=$? >> gpurun_out/final/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/final/gpu_tests.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/reference.json 2> gpurun_out/final/reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_reddit.csv python bench.py --workload reddit --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/final/ncu_launch.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_primitives.py -q -x -k "edge_sum and hub or spmm_q8 or weighted and hub" > gpurun_out/final/memcheck_prims.log 2>&1; echo rc=$? >> gpurun_out/final/memcheck_prims.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_layer.py -q -x -k "v6_h4_c7 or v6_noself" > gpurun_out/final/memcheck_v6.log 2>&1; echo rc=$? >> gpurun_out/final/memcheck_v6.log
