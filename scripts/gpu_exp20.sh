set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build20.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/sector_ubench scripts/sector_ubench.cu
UBENCH_FLAVOURS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none \
    -k regex:k_flavour --csv scripts/sector_ubench 2 320 > gpurun_out/ncu_ubench_320.csv 2>&1
UBENCH_FLAVOURS=1 timeout 300 scripts/sector_ubench 2 320 > gpurun_out/ubench_320.jsonl 2>&1
bash scripts/exp_env.sh friendster gpurun_out/exp_fr_layout.jsonl "GEER_ARC_POLICY=4" "GEER_ARC_POLICY=0" "GEER_WALK_LAYOUT=cols GEER_ARC_POLICY=4" > gpurun_out/exp_fr.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu -k "tiny or dense or split or rmat20_parity_full or ytable or layouts" > gpurun_out/gpu_tests_20.log 2>&1
