mkdir -p gpurun_out/r2g
python tools/l2q.py > gpurun_out/r2g/attrs.txt 2>&1 || python -c "
from cuda import cudart
for a in ('cudaDevAttrMaxPersistingL2CacheSize','cudaDevAttrL2CacheSize','cudaDevAttrMaxSharedMemoryPerMultiprocessor'):
    print(a, cudart.cudaDeviceGetAttribute(getattr(cudart.cudaDeviceAttr,a),0))" >> gpurun_out/r2g/attrs.txt 2>&1
run() { timeout 600 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2g/$1.json 2> gpurun_out/r2g/$1.err; }
run base
TANGO_EXP_NOSCATTER=1 run noscatter
TANGO_L2_PERSIST=1 run persist_normal
TANGO_L2_PERSIST=1 TANGO_L2_MISS_STREAMING=1 run persist_stream
