#!/bin/bash
# A/B of library variants (scripts/build_variant.py -> _varlib/<name>.so) on one box: per variant
# and config, a short bench line and an ncu launch list of one step.
# Usage: bash scripts/ab_launch.sh "<configs>" <name> [<name> ...]
CFGS=$1; shift
mkdir -p gpurun_out
for CFG in $CFGS; do
  for V in "$@"; do
    L=$PWD/_varlib/$V.so; [ "$V" = cur ] && L=$PWD/paper_2312_06123_b200/libgeer.so
    GEER_LIB=$L timeout 900 python bench.py --config $CFG --steps 3 --warmup 2 --no-cpu-baseline --no-spmm --no-accuracy \
        > gpurun_out/ab_bench_${V}_$CFG.log 2>&1
    GEER_LIB=$L timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 800 --csv \
        --log-file gpurun_out/ab_launch_${V}_$CFG.csv python bench.py --config $CFG --steps 1 --warmup 1 \
        --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ab_ncu_${V}_$CFG.log 2>&1
  done
done
