# round-2 baseline on the metric's config (Reddit-shaped layer): bench, launch list, ncu of the hub kernels, oracle timing
mkdir -p gpurun_out/r2a
nproc > gpurun_out/r2a/nproc.txt; lscpu | head -20 > gpurun_out/r2a/lscpu.txt
( time timeout 900 python bench.py --workload reddit --steps 5 --warmup 3 --no-cpu-baseline --layer-only --profile-breakdown > gpurun_out/r2a/bench_reddit.json 2> gpurun_out/r2a/bench_reddit.err ) 2> gpurun_out/r2a/time.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_src4|k_fwd_agg4|k_bwd_dst1_v4|k_fwd_stats2|k_fwd_alpha3|k_bwd_dst2|k_fwd_stats_t|k_gemm" -c 14 -o gpurun_out/r2a/reddit_full python bench.py --workload reddit --steps 1 --warmup 3 --no-cpu-baseline --layer-only > gpurun_out/r2a/ncu.log 2>&1
( time timeout 900 python -c "
import sys,time; sys.path.insert(0,'.')
from oracle import oracle as O; from paper_2308_00890_b200 import inputs
O.build(); g=inputs.workload_graph('reddit'); F,H,D=602,4,128
Hx=inputs.features(g.n,F); W,a,b=inputs.gat_params(F,H,D); dH=inputs.grad_out(g.n,H*D)
t=time.perf_counter(); f=O.gat_fwd(g,Hx,W,a,b,H,D,step=0); t1=time.perf_counter(); O.gat_bwd(g,f,Hx,W,a,b,dH); t2=time.perf_counter()
print('threads',O.num_threads(),'fwd',t1-t,'bwd',t2-t1)
" > gpurun_out/r2a/oracle_reddit.log 2>&1 ) 2>> gpurun_out/r2a/oracle_reddit.log
