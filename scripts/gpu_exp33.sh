set -x
mkdir -p gpurun_out
B="--steps 3 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy"
(cd _diagA && timeout 900 python bench.py $B > ../gpurun_out/d33_A.log 2>&1)
timeout 900 python bench.py $B > gpurun_out/d33_new.log 2>&1
