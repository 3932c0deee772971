python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_k9.log 2>&1
CFG=lj_full
timeout 900 ncu --set full --clock-control none -k regex:k_spmm_rows -s 3 -c 1 -f -o gpurun_out/spmm16_$CFG python scripts/spmm_probe.py $CFG > gpurun_out/ncu_spmm16_$CFG.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_spmm_rows -s 11 -c 1 -f -o gpurun_out/spmm64_$CFG python scripts/spmm_probe.py $CFG > gpurun_out/ncu_spmm64_$CFG.log 2>&1
python scripts/ncu_summary.py spmm gpurun_out/spmm16_$CFG.ncu-rep $CFG 16 > gpurun_out/ncu_k_spmm_q16_$CFG.json 2>/dev/null
python scripts/ncu_summary.py spmm gpurun_out/spmm64_$CFG.ncu-rep $CFG 64 > gpurun_out/ncu_k_spmm_q64_$CFG.json 2>/dev/null
timeout 1200 python bench.py > gpurun_out/bench_lj_k9.log 2>&1
timeout 600 python bench.py --config rmat20 > gpurun_out/bench_rmat20_k9.log 2>&1
