set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_$tag.log 2>&1; }
run def
run hash GEER_YTABLE=hash
run np2 GEER_WALK_NP=2
run np2m3 GEER_WALK_NP=2 GEER_WALK_MINB=3
run ov GEER_AMC_OVERLAP=1
run s32 GEER_WALK_SMEM_KB=32
run s16 GEER_WALK_SMEM_KB=16
tail -3 gpurun_out/gpu_tests.log
