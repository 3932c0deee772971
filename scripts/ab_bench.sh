#!/bin/bash
# Interleaved short bench lines of library variants on one box (GEER_LIB=_varlib/<name>.so).
# Usage: bash scripts/ab_bench.sh <config> <rounds> <name> [<name> ...]  -> gpurun_out/abb_<config>.jsonl
CFG=$1; R=$2; shift 2
mkdir -p gpurun_out
for r in $(seq 1 $R); do
  for V in "$@"; do
    GEER_LIB=$PWD/_varlib/$V.so timeout 900 python bench.py --config $CFG --steps 3 --warmup 2 --no-cpu-baseline \
        --no-spmm --no-accuracy 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); ph=d['phases_ms_per_step']
print(json.dumps({'variant':'$V','round':$r,'value':d['value'],'ms':d['ms_per_step'],'head':ph['smm_head'],'walks':ph['walks']}))" >> gpurun_out/abb_$CFG.jsonl
  done
done
