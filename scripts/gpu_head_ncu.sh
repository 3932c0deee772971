#!/bin/bash
# ncu --set full of the SMM head kernels (push + y-table build) on one config: one capture per
# kernel name of the first step (the head is the same in every step).
# Usage: bash scripts/gpu_head_ncu.sh <config> [tag]
CFG=${1:-lj_full}; TAG=${2:-head}
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_bkt_reduce_warp|k_bkt_scatter|k_bkt_count|k_bkt_reduce$|k_bkt_gather|k_yinsert|k_ybits|k_ywid|k_yrank' \
  -c 14 -f -o gpurun_out/${TAG}_$CFG python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline --no-spmm \
  --no-accuracy > gpurun_out/ncu_${TAG}_$CFG.log 2>&1
