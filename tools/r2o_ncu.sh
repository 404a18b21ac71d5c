mkdir -p gpurun_out/r2o
TANGO_L2_FETCH=32 timeout 1200 ncu --set full --clock-control none -k regex:"k2_bdst|k2_bsrc2|k2_fstats" -c 5 -o /tmp/ncu_light python bench.py --workload reddit --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2o/ncu.log 2>&1
python tools/ncu_stalls.py /tmp/ncu_light.ncu-rep > gpurun_out/r2o/stalls.txt 2>&1
python tools/ncu_summary.py /tmp/ncu_light.ncu-rep > gpurun_out/r2o/summary.txt 2>&1
ncu -i /tmp/ncu_light.ncu-rep --page raw --csv --metrics lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,dram__sectors_read.sum,lts__t_requests_srcunit_tex_op_read.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__d_sectors_fill_sysmem.sum,lts__d_sectors_fill_device.sum > gpurun_out/r2o/mem.csv 2>&1
