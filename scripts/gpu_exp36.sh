set -x
mkdir -p gpurun_out
B="--steps 3 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy"
(cd _diagA && timeout 900 python bench.py $B > ../gpurun_out/b36_noy.log 2>&1)
(cd _diagA && GEER_WALK_LAYOUT=cols24 timeout 900 python bench.py $B > ../gpurun_out/b36_noy_c24.log 2>&1)
CFG=lj_full
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_walks -s 5 -c 1 -f \
      -o gpurun_out/walks36_$CFG python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-spmm \
      --no-accuracy > gpurun_out/ncu_walks36_$CFG.log 2>&1
