set -x
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/sector_ubench scripts/sector_ubench.cu
UBENCH_FLAVOURS=1 timeout 300 scripts/sector_ubench 17 64,1024,16384 > gpurun_out/ubench_flavours.jsonl 2>&1
UBENCH_FLAVOURS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum --clock-control none -k regex:k_flavour --csv scripts/sector_ubench 17 16384 > gpurun_out/ncu_flavours.csv 2>&1
python __graft_entry__.py build > gpurun_out/build4.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu -k "tiny or dense or abi or spmm or fig3 or complete or lanczos" > gpurun_out/gpu_tests_push.log 2>&1
