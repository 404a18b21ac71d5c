mkdir -p gpurun_out
( time TANGO_FULL_PRODUCTS=1 timeout 2400 python -m pytest tests/test_gpu_fullsize.py -k products -x -q -s > gpurun_out/products_parity.log 2>&1 ) 2>> gpurun_out/products_parity.log
echo rc=$? >> gpurun_out/products_parity.log
free -g >> gpurun_out/products_parity.log
