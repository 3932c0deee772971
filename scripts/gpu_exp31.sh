set -x
mkdir -p gpurun_out
B="--steps 3 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy"
for i in 1 2; do
  (cd _cmp && timeout 900 python bench.py $B > ../gpurun_out/ab31_old_$i.log 2>&1)
  timeout 900 python bench.py $B > gpurun_out/ab31_new_$i.log 2>&1
done
