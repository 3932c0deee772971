set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
python scripts/dense_one.py 32 0.1 2 > gpurun_out/dense_one_32_2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmm_hub_exact -s 2 -c 1 -o gpurun_out/hub_exact python scripts/dense_one.py 32 0.1 2 > gpurun_out/hub_ncu.log 2>&1
tail -3 gpurun_out/hub_ncu.log
