# bench lines for the other BASELINE configs (one GPU): LJ-shaped 100k, Orkut-shaped 100k (eps 0.2 and 0.1)
set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python bench.py --config lj_full --queries 100000 --steps 3 --warmup 3 --no-spmm --no-cpu-baseline > gpurun_out/bench_cfg_lj.log 2>&1
timeout 900 python bench.py --config orkut_full --queries 100000 --eps 0.1 --steps 3 --warmup 3 --no-spmm --no-cpu-baseline > gpurun_out/bench_cfg_orkut01.log 2>&1
timeout 900 python bench.py --config orkut_full --queries 100000 --eps 0.2 --steps 3 --warmup 3 --no-spmm --no-cpu-baseline > gpurun_out/bench_cfg_orkut02.log 2>&1
for e in 0.5 0.2 0.05; do timeout 600 python bench.py --eps $e --steps 3 --warmup 3 --no-spmm --no-cpu-baseline > gpurun_out/bench_cfg_rmat20_$e.log 2>&1; done
for f in gpurun_out/bench_cfg_*.log; do echo $f; tail -1 $f | cut -c1-200; done
