mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:k_gemm_i8 -s 2 -c 1 -o gpurun_out/gemm8192 python tools/gemm_bench.py 8192 > gpurun_out/ncu_gemm.log 2>&1
