mkdir -p gpurun_out/r2m
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k2_fagg_seg|k2_bsrc1_seg" -c 2 -o /tmp/ncu_seg python bench.py --workload reddit --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2m/ncu.log 2>&1
python tools/ncu_stalls.py /tmp/ncu_seg.ncu-rep > gpurun_out/r2m/stalls.txt 2>&1
python tools/ncu_hot.py /tmp/ncu_seg.ncu-rep k2_fagg_seg > gpurun_out/r2m/hot_fagg_seg.txt 2>&1
python tools/ncu_hot.py /tmp/ncu_seg.ncu-rep k2_bsrc1_seg > gpurun_out/r2m/hot_bsrc1_seg.txt 2>&1
ncu -i /tmp/ncu_seg.ncu-rep -k regex:k2_fagg_seg --page source --csv --print-source sass > gpurun_out/r2m/src_fagg_seg.csv 2>&1
