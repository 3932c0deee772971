set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "tiny or rmat20_parity_full or layouts" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_$tag.log 2>&1; }
run def
run yef GEER_Y_EVICT_FIRST=1
run l2p GEER_L2_PERSIST=1
run both GEER_Y_EVICT_FIRST=1 GEER_L2_PERSIST=1
run ov GEER_AMC_OVERLAP=1
run ov_both GEER_AMC_OVERLAP=1 GEER_Y_EVICT_FIRST=1 GEER_L2_PERSIST=1
tail -3 gpurun_out/gpu_tests.log
