set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
for V in "2 3" "2 4" "1 4" "2 2" "1 3"; do set -- $V
  GEER_WALK_NP=$1 GEER_WALK_MINB=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_np$1_m$2.log 2>&1
done
GEER_AMC_OVERLAP=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_overlap.log 2>&1
GEER_WALK_SMEM_KB=32 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_smem32.log 2>&1
tail -3 gpurun_out/gpu_tests.log
