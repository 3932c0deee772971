set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build9.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bkt_reduce -s 2 -c 2 -f -o gpurun_out/bkt_reduce9 python bench.py --config rmat20 --steps 1 --warmup 1 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ncu_bkt9.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:geer:: -c 700 --csv --log-file gpurun_out/launches_lj_9.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ncu_launch9lj.log 2>&1
bash scripts/exp_env.sh lj_full gpurun_out/exp_policy2_lj.jsonl "GEER_ARC_POLICY=1" "GEER_ARC_POLICY=2" "GEER_Y_POLICY=2" "GEER_ARC_POLICY=2 GEER_Y_POLICY=2" "GEER_WALK_MINB=5" > gpurun_out/exp_policy2.log 2>&1
