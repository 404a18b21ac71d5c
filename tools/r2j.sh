# default bench + ncu captures of one layer step (reports kept in /tmp on the box, CSV summaries returned)
mkdir -p gpurun_out/r2j
( time timeout 1200 python bench.py > gpurun_out/r2j/bench.json 2> gpurun_out/r2j/bench.err ) 2> gpurun_out/r2j/bench_time.log
for w in reddit arxiv; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k2_|k_quantize" -c 12 -o /tmp/ncu_$w python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2j/ncu_$w.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_$w.ncu-rep > gpurun_out/r2j/ncu_$w.summary.txt 2>&1
  cp profiles/ncu_traffic.json /tmp/nt.json; python tools/ncu_to_traffic.py /tmp/ncu_$w.ncu-rep $w r2j_$w > gpurun_out/r2j/traffic_$w.json 2>&1
  for k in k2_fagg k2_bsrc1 k2_bdst_a k2_bsrc2; do python tools/ncu_hot.py /tmp/ncu_$w.ncu-rep $k > gpurun_out/r2j/hot_${w}_$k.txt 2>&1; done
done
cp profiles/ncu_traffic.json gpurun_out/r2j/ncu_traffic.json
