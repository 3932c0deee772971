#!/bin/bash
# k_seg_max2 read-before-atomicMax: parity suite + launch lists (k_seg_max2 time) + graded line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/m2_gpu_tests.log 2>&1; tail -1 gpurun_out/m2_gpu_tests.log
for CFG in orkut_full lj_full friendster; do
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 800 --csv \
      --log-file gpurun_out/m2_launches_$CFG.csv python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline \
      --no-spmm --no-accuracy > gpurun_out/m2_ncu_launch_$CFG.log 2>&1
  python tools_launches.py gpurun_out/m2_launches_$CFG.csv 40 1 | grep -E "k_first_wave|k_seg_max2|total"
done
timeout 1200 python bench.py > gpurun_out/m2_bench_lj.log 2>/dev/null; tail -1 gpurun_out/m2_bench_lj.log | cut -c1-200
timeout 1800 python bench.py --config friendster --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/m2_bench_friendster.log 2>/dev/null; tail -1 gpurun_out/m2_bench_friendster.log | cut -c1-200
