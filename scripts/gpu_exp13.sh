set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build14.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu -k "tiny or dense or split or rmat20_parity or lanczos" > gpurun_out/gpu_tests_14.log 2>&1
timeout 600 python bench.py --config rmat20 --steps 5 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/bench_rmat20_14.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_rmat20_14.csv python bench.py --config rmat20 --steps 2 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ncu_launch14.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/bench_lj_14.log 2>&1
