# quick check: parity subset + default bench (+ optional variants in $VARIANTS as "tag:ENV=V,ENV=V ...")
set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "${PYTEST_K:-tiny or rmat20_parity_full or layouts or query_ids}" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_$tag.log 2>&1; }
run def
for v in $VARIANTS; do tag=${v%%:*}; envs=${v#*:}; run $tag $(echo $envs | tr ',' ' '); done
tail -3 gpurun_out/gpu_tests.log
for f in gpurun_out/bench_*.log; do echo $f; tail -1 $f | cut -c1-120; done
