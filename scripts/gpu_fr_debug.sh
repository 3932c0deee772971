set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 900 python bench.py --config friendster --queries 125000 --steps 1 --warmup 1 --no-spmm --no-cpu-baseline > gpurun_out/fr_dbg.log 2>&1
tail -3 gpurun_out/fr_dbg.log
