# round bench: full GPU tests, bench (default config), ncu launch list, ncu --set full of k_walks
# (each ncu run preceded by the identical command without ncu)
set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-spmm"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1
CMD1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-spmm"
timeout 300 $CMD1 > gpurun_out/plain_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_walks" -s 5 -c 1 -o gpurun_out/prof_walks -f $CMD1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; tail -2 gpurun_out/bench.log | cut -c1-300
