set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build29.log 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests_29.log 2>&1
timeout 600 python bench.py --config rmat20 --steps 5 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/bench_rmat20_29.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/bench_lj_29.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file gpurun_out/launches_rmat20_29.csv python bench.py --config rmat20 --steps 1 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ncu_l29.log 2>&1
