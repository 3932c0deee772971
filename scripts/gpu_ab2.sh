set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "tiny or rmat20_parity_full or query_ids" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_$tag.log 2>&1; }
run v3_np_noov GEER_WALK_KERNEL=3 GEER_AMC_OVERLAP=0
run v3_np_ov GEER_WALK_KERNEL=3 GEER_AMC_OVERLAP=1
run v4np1_p_noov GEER_WALK_KERNEL=4 GEER_WALK_NP=1 GEER_WALK_MINB=4 GEER_WALK_SMEM_KB=24 GEER_AMC_OVERLAP=0 GEER_WALK_PERSIST=1
run v4np1_p_ov GEER_WALK_KERNEL=4 GEER_WALK_NP=1 GEER_WALK_MINB=4 GEER_WALK_SMEM_KB=24 GEER_AMC_OVERLAP=1 GEER_WALK_PERSIST=1
(cd _ab && python paper_2312_06123_b200/build.py > /dev/null 2>&1; timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > ../gpurun_out/bench_ab_old.log 2>&1)
tail -2 gpurun_out/gpu_tests.log
