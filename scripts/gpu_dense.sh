# dense-mode check: its tests, K9 tests, the timing probe, launch lists
set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_parity.py -m gpu -q -x -k "dense or k9 or tiny_parity" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python scripts/dense_probe.py > gpurun_out/dense_probe.jsonl 2> gpurun_out/dense_probe.err
for c in ${DENSE_CASES:-"1000 0.05 2" "32 0.1 2"}; do
  set -- $c
  python scripts/dense_one.py $1 $2 $3 > gpurun_out/dense_one_$1_$3.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dense_launch_$1_$3.csv python scripts/dense_one.py $1 $2 $3 > /dev/null 2>&1
done
tail -5 gpurun_out/gpu_tests.log
