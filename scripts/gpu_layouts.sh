# walk layouts: plain bench per layout, then one ncu pass (cheap metrics, no cache flush) over the
# timed step's k_walks launches per layout
set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "spmm" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
for L in packed cols arcs; do
  GEER_WALK_LAYOUT=$L timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_$L.log 2>&1
done
for L in packed cols; do
  GEER_WALK_LAYOUT=$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --cache-control none --clock-control none -k regex:k_walks -s 45 -c 15 --csv --log-file gpurun_out/walks_$L.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/ncu_$L.log 2>&1
done
tail -3 gpurun_out/gpu_tests.log
