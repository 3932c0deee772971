#!/bin/bash
# Final bench lines of the round (after gpu_final.sh's captures): all -m gpu tests, the graded
# line (full), config 1, Orkut- and Friendster-shaped lines.
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_lines.log 2>&1
tail -2 gpurun_out/gpu_tests_lines.log
timeout 1200 python bench.py > gpurun_out/bench_lj.log 2>&1
timeout 600 python bench.py --config rmat20 > gpurun_out/bench_rmat20.log 2>&1
timeout 900 python bench.py --config orkut_full --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_orkut.log 2>&1
timeout 2400 python bench.py --config friendster --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_friendster.log 2>&1
