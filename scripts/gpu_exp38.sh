set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build38.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu -k "layout or tiny or rmat20_parity_full or variants or split" > gpurun_out/gpu_tests_38.log 2>&1
rm -f gpurun_out/exp38.jsonl
bash scripts/exp_env.sh lj_full gpurun_out/exp38.jsonl "GEER_X=0" "GEER_WALK_LAYOUT=cols24" > gpurun_out/exp38.log 2>&1
bash scripts/exp_env.sh orkut_full gpurun_out/exp38.jsonl "GEER_X=0" "GEER_WALK_LAYOUT=cols24" "GEER_WALK_L2_KEEP=0" >> gpurun_out/exp38.log 2>&1
bash scripts/exp_env.sh rmat20 gpurun_out/exp38.jsonl "GEER_X=0" "GEER_WALK_LAYOUT=dord" >> gpurun_out/exp38.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file gpurun_out/launches_lj_38.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ncu_l38.log 2>&1
GEER_WALK_LAYOUT=cols24 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file gpurun_out/launches_lj_38c.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ncu_l38c.log 2>&1
