set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
(cd _ab && python paper_2312_06123_b200/build.py > /dev/null 2>&1)
export GEER_WALK_KERNEL=3 GEER_AMC_OVERLAP=0
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/plain_new.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_walks -s 15 -c 5 --csv --log-file gpurun_out/walks_new.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/ncu_new.log 2>&1
(cd _ab && timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > ../gpurun_out/plain_old.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_walks -s 15 -c 5 --csv --log-file ../gpurun_out/walks_old.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > ../gpurun_out/ncu_old.log 2>&1)
