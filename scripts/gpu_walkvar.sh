set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
for M in 4 3; do
  GEER_WALK_MINB=$M timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_m$M.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors.sum --cache-control none --clock-control none -k regex:k_walks -s 45 -c 15 --csv --log-file gpurun_out/walks_m4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/ncu_m4.log 2>&1
timeout 300 python scripts/spmm_probe.py > gpurun_out/spmm_probe.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active --cache-control none --clock-control none -k regex:spmm --csv --log-file gpurun_out/spmm_launches.csv python scripts/spmm_probe.py > gpurun_out/ncu_spmm.log 2>&1
tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/spmm_probe.log
