set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build34.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu -k "layout or tiny or rmat20_parity_full or split or full_size or variants" > gpurun_out/gpu_tests_34.log 2>&1
B="--steps 3 --warmup 3 --no-cpu-baseline --no-spmm --no-accuracy"
timeout 900 python bench.py $B > gpurun_out/b34_lj_dord.log 2>&1
GEER_WALK_LAYOUT=cols24 timeout 900 python bench.py $B > gpurun_out/b34_lj_c24.log 2>&1
timeout 900 python bench.py --config rmat20 $B > gpurun_out/b34_r20_packed.log 2>&1
GEER_WALK_LAYOUT=dord timeout 900 python bench.py --config rmat20 $B > gpurun_out/b34_r20_dord.log 2>&1
timeout 900 python bench.py --config orkut_full $B > gpurun_out/b34_ork_dord.log 2>&1
