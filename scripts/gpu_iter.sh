#!/bin/bash
# One build -> measure iteration on a GPU box: all -m gpu tests, short bench lines of the graded
# config and config 1 (no cpu_baseline / K9 / accuracy legs), ncu launch lists of both.
# Usage: bash scripts/gpu_iter.sh [tag]
TAG=${1:-it}
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build_$TAG.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests_$TAG.log 2>&1
tail -2 gpurun_out/gpu_tests_$TAG.log
for CFG in lj_full rmat20; do
  timeout 900 python bench.py --config $CFG --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/bench_${TAG}_$CFG.log 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 800 --csv \
      --log-file gpurun_out/launches_${TAG}_$CFG.csv python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline \
      --no-spmm --no-accuracy > gpurun_out/ncu_launch_${TAG}_$CFG.log 2>&1
done
