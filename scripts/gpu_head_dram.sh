#!/bin/bash
# DRAM bytes of the SMM head kernels of one step (bench.py --steps 1 --warmup 0) -> launch list CSV.
CFG=${1:-lj_full}
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k 'regex:^k_(bkt|y|first_wave|compact|seg|ent_deg|decide|scan|query_pairs|setup|flag_phase|init_frontier|dense)' \
    --csv --log-file gpurun_out/head_dram_$CFG.csv python bench.py --config $CFG --steps 1 --warmup 0 \
    --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/head_dram_$CFG.log 2>&1
