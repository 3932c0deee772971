set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
GEER_WALK_KERNEL=4 GEER_WALK_NP=1 timeout 900 python -m pytest tests -m gpu -x -q -k "tiny or rmat20_parity_full" > gpurun_out/gpu_tests_v4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_v4.log
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_$tag.log 2>&1; }
run v3 GEER_WALK_KERNEL=3
run v3_noov GEER_WALK_KERNEL=3 GEER_AMC_OVERLAP=0
run v4np1 GEER_WALK_KERNEL=4 GEER_WALK_NP=1 GEER_WALK_MINB=4 GEER_WALK_SMEM_KB=24
run v4np2 GEER_WALK_KERNEL=4 GEER_WALK_NP=2 GEER_WALK_MINB=4 GEER_WALK_SMEM_KB=24
run v4np1_noov GEER_WALK_KERNEL=4 GEER_WALK_NP=1 GEER_WALK_MINB=4 GEER_WALK_SMEM_KB=24 GEER_AMC_OVERLAP=0
tail -3 gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests_v4.log
