set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build16.log 2>&1
bash scripts/exp_env.sh lj_full gpurun_out/exp_y64_lj.jsonl "GEER_ARC_POLICY=4" "GEER_ARC_POLICY=4 GEER_Y_POLICY=4" "GEER_ARC_POLICY=4 GEER_Y_POLICY=6" "GEER_ARC_POLICY=4 GEER_Y_POLICY=5" "GEER_ARC_POLICY=1" > gpurun_out/exp_y64.log 2>&1
bash scripts/exp_env.sh orkut_full gpurun_out/exp_y64_orkut.jsonl "GEER_ARC_POLICY=0" "GEER_ARC_POLICY=1" "GEER_ARC_POLICY=4" "GEER_ARC_POLICY=4 GEER_Y_POLICY=4" > gpurun_out/exp_y64o.log 2>&1
