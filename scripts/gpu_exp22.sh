set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build22.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu -k "layouts or tiny_parity_and_exact or rmat20_parity_full or ytable" > gpurun_out/gpu_tests_22.log 2>&1
bash scripts/exp_env.sh lj_full gpurun_out/exp_c24_lj.jsonl "GEER_WALK_LAYOUT=cols24" "GEER_WALK_LAYOUT=cols" > gpurun_out/exp_c24.log 2>&1
bash scripts/exp_env.sh orkut_full gpurun_out/exp_c24_orkut.jsonl "GEER_WALK_LAYOUT=cols24" "GEER_WALK_LAYOUT=cols" > gpurun_out/exp_c24o.log 2>&1
