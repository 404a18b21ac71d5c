mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:"k_bwd_src4|k_bwd_src_combine|k_fwd_agg4|k_fwd_combine" -c 5 -o gpurun_out/pass_final python bench.py --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/ncu_pass.log 2>&1
