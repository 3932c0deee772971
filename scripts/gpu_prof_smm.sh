# ncu --set full of the SMM-head kernels of one timed step (k_yinsert, k_run_reduce, k_seg_max2)
set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
CMD1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-spmm"
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_$tag.log 2>&1; }
run cols GEER_WALK_LAYOUT=cols
run arcs GEER_WALK_LAYOUT=arcs
timeout 300 $CMD1 > gpurun_out/plain_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_yinsert|k_run_reduce|k_seg_max2" -s 6 -c 6 -o gpurun_out/prof_smm -f $CMD1 > gpurun_out/ncu_smm.log 2>&1
for f in gpurun_out/bench_*.log; do echo $f; tail -1 $f | cut -c1-120; done
