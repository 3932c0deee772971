#!/bin/bash
# K9 A/B on one box: scripts/spmm_ab.py (q = 16 / 64, L2 flushed) for library variants
# (scripts/build_variant.py -> _varlib/<name>.so; "cur" = the in-tree build), two passes.
# Usage: bash scripts/k9_ab.sh "<configs>" <name> [<name> ...]
CFGS=$1; shift
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/k9_build.log 2>&1 || exit 1
for CFG in $CFGS; do
for pass in 1 2; do
for V in "$@"; do
  L=$PWD/_varlib/$V.so; [ "$V" = cur ] && L=$PWD/paper_2312_06123_b200/libgeer.so
  GEER_LIB=$L timeout 600 python scripts/spmm_ab.py $CFG >> gpurun_out/k9_ab.jsonl 2>> gpurun_out/k9_ab.err
done
done
done
