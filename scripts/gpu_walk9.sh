set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "tiny or rmat20_parity_full or query_ids" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
GEER_WALK_KERNEL=4 GEER_WALK_NP=1 timeout 900 python -m pytest tests -m gpu -x -q -k "tiny or rmat20_parity_full" > gpurun_out/gpu_tests_v4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_v4.log
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_$tag.log 2>&1; }
run v3_np_noov GEER_WALK_KERNEL=3 GEER_AMC_OVERLAP=0
run v3_np_ov GEER_WALK_KERNEL=3 GEER_AMC_OVERLAP=1
run v4np1_np_noov GEER_WALK_KERNEL=4 GEER_WALK_NP=1 GEER_WALK_MINB=4 GEER_WALK_SMEM_KB=24 GEER_AMC_OVERLAP=0
run v4np1_np_ov GEER_WALK_KERNEL=4 GEER_WALK_NP=1 GEER_WALK_MINB=4 GEER_WALK_SMEM_KB=24 GEER_AMC_OVERLAP=1
run v4np2_np_noov GEER_WALK_KERNEL=4 GEER_WALK_NP=2 GEER_WALK_MINB=4 GEER_WALK_SMEM_KB=24 GEER_AMC_OVERLAP=0
run v4np1_np_noov_s48 GEER_WALK_KERNEL=4 GEER_WALK_NP=1 GEER_WALK_MINB=4 GEER_WALK_SMEM_KB=48 GEER_AMC_OVERLAP=0
run v4np1_p_noov GEER_WALK_KERNEL=4 GEER_WALK_NP=1 GEER_WALK_MINB=4 GEER_WALK_SMEM_KB=24 GEER_AMC_OVERLAP=0 GEER_WALK_PERSIST=1
python -c "
import sys,time; sys.path.insert(0,'.')
import workloads as W
t=time.time(); g,p,_=W.load_config('lj_full'); print('lj_full', g.n, g.nnz, g.degrees().max(), round(time.time()-t,1), flush=True)
t=time.time(); g,p,_=W.load_config('orkut_full'); print('orkut_full', g.n, g.nnz, g.degrees().max(), round(time.time()-t,1), flush=True)
" > gpurun_out/gen.log 2>&1
tail -3 gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests_v4.log; cat gpurun_out/gen.log
