set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build21.log 2>&1
bash scripts/exp_env.sh lj_full gpurun_out/exp_noy_lj.jsonl "GEER_Y_POLICY=0" "GEER_Y_POLICY=8" > gpurun_out/exp_noy.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_lj_21.log 2>&1
timeout 600 python bench.py --config rmat20 > gpurun_out/bench_rmat20_21.log 2>&1
