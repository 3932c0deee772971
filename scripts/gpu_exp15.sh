set -x
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/sector_ubench scripts/sector_ubench.cu
UBENCH_FLAVOURS=1 timeout 300 scripts/sector_ubench 17 64,1024,16384 > gpurun_out/ubench_flavours2.jsonl 2>&1
UBENCH_FLAVOURS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum --clock-control none -k regex:k_flavour --csv scripts/sector_ubench 17 16384 > gpurun_out/ncu_flavours2.csv 2>&1
python __graft_entry__.py build > gpurun_out/build15.log 2>&1
bash scripts/exp_env.sh lj_full gpurun_out/exp_l264_lj.jsonl "GEER_ARC_POLICY=1" "GEER_ARC_POLICY=3" "GEER_ARC_POLICY=4" > gpurun_out/exp_l264.log 2>&1
