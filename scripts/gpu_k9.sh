set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "spmm" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python scripts/spmm_probe.py > gpurun_out/spmm_probe.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active --cache-control none --clock-control none -k regex:spmm -c 4 --csv --log-file gpurun_out/spmm_launches.csv python scripts/spmm_probe.py > gpurun_out/ncu_spmm.log 2>&1
tail -2 gpurun_out/gpu_tests.log; cat gpurun_out/spmm_probe.log
