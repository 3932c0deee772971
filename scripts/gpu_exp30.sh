set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build30.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "layout or tiny or rmat20_parity_full or split or full_size" > gpurun_out/gpu_tests_30.log 2>&1
for i in 1 2; do timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/bench_lj_30_$i.log 2>&1; done
timeout 900 python bench.py --config orkut_full --steps 3 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/bench_orkut_30.log 2>&1
nvidia-smi -q -d POWER,CLOCK > gpurun_out/smi30.txt 2>&1
