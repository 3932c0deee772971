set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
for v in ${CFG_VARIANTS:-"def:"}; do
  tag=${v%%:*}; envs=${v#*:}
  env $(echo $envs | tr ',' ' ') timeout 900 python bench.py --config ${CFG:-lj_full} --queries ${NQ:-100000} --eps ${EPS:-0.1} --steps 2 --warmup 3 --no-spmm --no-cpu-baseline > gpurun_out/bench_cv_$tag.log 2>&1
done
