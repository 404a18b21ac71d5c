# P1 writes full-sector {∂α, signed α} records at in-CSR slots (TANGO_P2_REC default on): parity of all
# variants, Reddit layer rec vs gather (interleaved, twice), ncu of P1 / P2 with records
mkdir -p gpurun_out/r3c
timeout 1800 python -m pytest tests/test_gpu_layer.py -x -q > gpurun_out/r3c/tests.log 2>&1; echo rc=$? >> gpurun_out/r3c/tests.log
for i in 1 2; do
timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3c/rec$i.json 2> gpurun_out/r3c/rec$i.err
TANGO_P2_REC=0 timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3c/gather$i.json 2> gpurun_out/r3c/gather$i.err
done
timeout 1200 ncu --set full --clock-control none -k regex:"k2_bsrc1_seg|k2_bdst" -c 3 -o /tmp/ncu_c python bench.py --workload reddit --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r3c/ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu_c.ncu-rep > gpurun_out/r3c/ncu_summary.txt 2>&1
