mkdir -p gpurun_out
for v in 1 0.5 0.25 0.125 1 0.25; do
  TANGO_DW_CTAS_PER_SM=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --layer-only 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],4), d['kernel_ms_per_step'].get('gemm_splitk_i64'))" >> gpurun_out/dw.log
done
