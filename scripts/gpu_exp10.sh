set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build10.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu -k "tiny or dense or split or rmat20_parity_full or lanczos" > gpurun_out/gpu_tests_10.log 2>&1
timeout 600 python bench.py --config rmat20 --steps 5 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/bench_rmat20_10.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_rmat20_10.csv python bench.py --config rmat20 --steps 2 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ncu_launch10.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c 700 --csv --log-file gpurun_out/launches_lj_10.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ncu_launch10lj.log 2>&1
