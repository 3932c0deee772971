set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
for v in "def:" "np2m3:GEER_WALK_NP=2,GEER_WALK_MINB=3" "np2m4:GEER_WALK_NP=2,GEER_WALK_MINB=4"; do
  tag=${v%%:*}; envs=${v#*:}
  env $(echo $envs | tr ',' ' ') timeout 900 python bench.py --config lj_full --queries 100000 --steps 2 --warmup 3 --no-spmm --no-cpu-baseline > gpurun_out/bench_lj_$tag.log 2>&1
done
