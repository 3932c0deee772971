set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
CMD1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-spmm"
timeout 300 $CMD1 > gpurun_out/plain_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_run_reduce|k_emit|k_seg_max2" -s 6 -c 3 -o gpurun_out/prof_head -f $CMD1 > gpurun_out/ncu_head.log 2>&1
tail -2 gpurun_out/ncu_head.log
