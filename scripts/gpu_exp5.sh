set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build5.log 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests_5.log 2>&1
timeout 600 python bench.py --config rmat20 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_rmat20_5.log 2>&1
bash scripts/exp_env.sh lj_full gpurun_out/exp_layout_lj.jsonl "GEER_WALK_LAYOUT=arcs" "GEER_WALK_LAYOUT=cols" "GEER_WALK_LAYOUT=cols GEER_WALK_TILES=0" "GEER_WALK_LAYOUT=cols GEER_ARC_POLICY=1" > gpurun_out/exp_layout.log 2>&1
