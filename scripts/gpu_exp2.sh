set -x
mkdir -p gpurun_out
bash scripts/exp_env.sh lj_full gpurun_out/exp_policy_lj.jsonl "GEER_ARC_POLICY=0" "GEER_ARC_POLICY=1" "GEER_ARC_POLICY=2" "GEER_ARC_POLICY=1 GEER_Y_POLICY=2" "GEER_ARC_POLICY=2 GEER_Y_POLICY=2" "GEER_Y_POLICY=2" > gpurun_out/exp_policy.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/sector_ubench scripts/sector_ubench.cu
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:k_independent --csv scripts/sector_ubench 17 64,1024,16384 > gpurun_out/ncu_ubench.csv 2> gpurun_out/ncu_ubench.err
