set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
(cd _ab && python paper_2312_06123_b200/build.py > /dev/null 2>&1; timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > ../gpurun_out/bench_ab_old.log 2>&1)
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_$tag.log 2>&1; }
run v3_np_noov GEER_WALK_KERNEL=3 GEER_AMC_OVERLAP=0
run v4np1_p_noov GEER_WALK_KERNEL=4 GEER_WALK_NP=1 GEER_WALK_MINB=4 GEER_WALK_SMEM_KB=24 GEER_AMC_OVERLAP=0 GEER_WALK_PERSIST=1
(cd _ab && timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > ../gpurun_out/bench_ab_old2.log 2>&1)
GEER_WALK_KERNEL=4 GEER_WALK_NP=1 GEER_WALK_MINB=4 GEER_WALK_SMEM_KB=24 GEER_AMC_OVERLAP=0 GEER_WALK_PERSIST=1 timeout 600 python bench.py --config lj_full --queries 100000 --steps 2 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_lj.log 2>&1
for f in gpurun_out/bench_*.log; do echo $f; tail -1 $f | cut -c1-150; done
