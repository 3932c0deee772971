set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build6.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_rmat20_push.csv python bench.py --config rmat20 --steps 2 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ncu_launch6.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_bkt_reduce -s 2 -c 2 -f -o gpurun_out/bkt_reduce python bench.py --config rmat20 --steps 1 --warmup 1 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ncu_bkt.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "lanczos or split" > gpurun_out/gpu_tests_6.log 2>&1
