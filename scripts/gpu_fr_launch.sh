set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
CMD="python bench.py --config friendster --queries 125000 --steps 1 --warmup 1 --no-spmm --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/fr_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fr_launches.csv $CMD > gpurun_out/fr_ncu.log 2>&1
tail -2 gpurun_out/fr_ncu.log
