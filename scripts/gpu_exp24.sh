set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build25.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu -k "tiny or dense or split or rmat20_parity or layouts or ytable" > gpurun_out/gpu_tests_25.log 2>&1
for i in 1 2; do timeout 600 python bench.py --config rmat20 --steps 5 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/bench_rmat20_25_$i.log 2>&1; done
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/bench_lj_25.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 600 --csv --log-file gpurun_out/launches_rmat20_25.csv python bench.py --config rmat20 --steps 2 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ncu_launch25.log 2>&1
