set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build12.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bkt_reduce_warp -s 2 -c 1 -f -o gpurun_out/bkt_warp12 python bench.py --config rmat20 --steps 1 --warmup 1 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ncu_bkt12.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_yhash -s 0 -c 1 -f -o gpurun_out/yhash12 python bench.py --config rmat20 --steps 1 --warmup 1 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ncu_yhash12.log 2>&1
