#!/bin/bash
# K9 refresh on one box: all -m gpu tests; ncu --set full of K9 at q = 16 / 64 on the graded
# config and config 1 (-> profiles/ncu_k_spmm_q*_<cfg>_r02.json, read by bench.py); bench lines.
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_k9.log 2>&1
tail -2 gpurun_out/gpu_tests_k9.log
for CFG in lj_full rmat20; do
timeout 900 ncu --set full --clock-control none -k 'regex:k_spmm_(rows|items)' -s 3 -c 1 -f -o gpurun_out/spmm16_$CFG python scripts/spmm_probe.py $CFG > gpurun_out/ncu_spmm16_$CFG.log 2>&1
timeout 900 ncu --set full --clock-control none -k 'regex:k_spmm_(rows|items)' -s 11 -c 1 -f -o gpurun_out/spmm64_$CFG python scripts/spmm_probe.py $CFG > gpurun_out/ncu_spmm64_$CFG.log 2>&1
python scripts/ncu_summary.py spmm gpurun_out/spmm16_$CFG.ncu-rep $CFG 16 > gpurun_out/ncu_k_spmm_q16_$CFG.json 2>gpurun_out/ncu_sum16_$CFG.err
python scripts/ncu_summary.py spmm gpurun_out/spmm64_$CFG.ncu-rep $CFG 64 > gpurun_out/ncu_k_spmm_q64_$CFG.json 2>gpurun_out/ncu_sum64_$CFG.err
done
