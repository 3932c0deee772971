set -x
mkdir -p gpurun_out
B="--steps 3 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy"
timeout 900 python bench.py $B > gpurun_out/d32_new.log 2>&1
(cd _diagA && timeout 900 python bench.py $B > ../gpurun_out/d32_A.log 2>&1)
(cd _diagC && timeout 900 python bench.py $B > ../gpurun_out/d32_C.log 2>&1)
