set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build37.log 2>&1
rm -f gpurun_out/exp37.jsonl
bash scripts/exp_env.sh lj_full gpurun_out/exp37.jsonl "GEER_WALK_L2_KEEP=0" "GEER_WALK_L2_KEEP=0.15" "GEER_WALK_L2_KEEP=0.3" "GEER_WALK_L2_KEEP=0.45" "GEER_WALK_L2_KEEP=0.6" "GEER_WALK_L2_KEEP=0.3 GEER_WALK_LAYOUT=cols24" "GEER_WALK_L2_KEEP=0 GEER_WALK_LAYOUT=cols24" > gpurun_out/exp37.log 2>&1
