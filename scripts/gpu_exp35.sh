set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build35.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu -k "layout or tiny or rmat20_parity_full or variants" > gpurun_out/gpu_tests_35.log 2>&1
B="--steps 3 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy"
timeout 900 python bench.py $B > gpurun_out/b35_lj_dord.log 2>&1
GEER_WALK_LAYOUT=cols24 timeout 900 python bench.py $B > gpurun_out/b35_lj_c24.log 2>&1
GEER_WALK_LAYOUT=dord timeout 900 python bench.py --config rmat20 $B > gpurun_out/b35_r20_dord.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file gpurun_out/launches_lj_35.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ncu_l35.log 2>&1
