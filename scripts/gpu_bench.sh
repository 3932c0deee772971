# round bench: GPU tests, bench (default config), ncu launch list, ncu --set full of k_walks
set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/ncu.log 2>&1
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/plain_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_walks" -s 20 -c 1 -o gpurun_out/prof_walks -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/ncu_full.log 2>&1
timeout 300 python scripts/spmm_probe.py > gpurun_out/spmm_probe.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_spmm_rows" -s 2 -c 1 -o gpurun_out/prof_spmm -f python scripts/spmm_probe.py > gpurun_out/ncu_full_spmm.log 2>&1
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/bench.log
