set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "spmm or tiny" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_$tag.log 2>&1; }
run h0_np1_m3 GEER_WALK_HINTS=0 GEER_WALK_NP=1 GEER_WALK_MINB=3
run h3_np1_m3 GEER_WALK_HINTS=3 GEER_WALK_NP=1 GEER_WALK_MINB=3
run h1_np1_m3 GEER_WALK_HINTS=1 GEER_WALK_NP=1 GEER_WALK_MINB=3
run h0_np1_m4_s24 GEER_WALK_HINTS=0 GEER_WALK_NP=1 GEER_WALK_MINB=4 GEER_WALK_SMEM_KB=24
run h0_np1_m4_s32 GEER_WALK_HINTS=0 GEER_WALK_NP=1 GEER_WALK_MINB=4 GEER_WALK_SMEM_KB=32
run h0_np2_m3 GEER_WALK_HINTS=0 GEER_WALK_NP=2 GEER_WALK_MINB=3
run h0_np2_m4_s24 GEER_WALK_HINTS=0 GEER_WALK_NP=2 GEER_WALK_MINB=4 GEER_WALK_SMEM_KB=24
run h0_np2_m2 GEER_WALK_HINTS=0 GEER_WALK_NP=2 GEER_WALK_MINB=2
tail -3 gpurun_out/gpu_tests.log
