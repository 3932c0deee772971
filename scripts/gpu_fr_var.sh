set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
for v in ${FR_VARIANTS:-"def:"}; do
  tag=${v%%:*}; envs=${v#*:}
  env $(echo $envs | tr ',' ' ') timeout 900 python bench.py --config friendster --queries 125000 --steps 2 --warmup 3 --no-spmm --no-cpu-baseline > gpurun_out/bench_fr_$tag.log 2>&1
done
