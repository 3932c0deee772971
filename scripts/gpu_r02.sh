#!/bin/bash
# Round-2 GPU session driver: roofline ubench, graded bench line, ncu of K6 / K9 on the graded config.
# Usage (from the repo root, on the GPU box): bash scripts/gpu_r02.sh [config]
set -x
CFG=${1:-lj_full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt
python __graft_entry__.py build > gpurun_out/build.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/sector_ubench scripts/sector_ubench.cu
timeout 300 scripts/sector_ubench 32 > gpurun_out/sector_ubench.jsonl 2> gpurun_out/sector_ubench.err
timeout 900 python bench.py --config $CFG --steps 5 --warmup 3 > gpurun_out/bench_$CFG.log 2>&1
timeout 600 python scripts/walk_batch_steps.py $CFG > gpurun_out/walk_steps_$CFG.json 2> gpurun_out/walk_steps_$CFG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_walks -s 5 -c 1 -f \
    -o gpurun_out/walks_$CFG python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-spmm \
    --no-accuracy > gpurun_out/ncu_walks_$CFG.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_spmm_rows -s 3 -c 1 -f -o gpurun_out/spmm16_$CFG \
    python scripts/spmm_probe.py $CFG > gpurun_out/ncu_spmm16_$CFG.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_spmm_rows -s 11 -c 1 -f -o gpurun_out/spmm64_$CFG \
    python scripts/spmm_probe.py $CFG > gpurun_out/ncu_spmm64_$CFG.log 2>&1
ls -la gpurun_out
