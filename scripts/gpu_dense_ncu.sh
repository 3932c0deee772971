set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
for c in "1000 0.05 2" "1000 0.05 1" "32 0.1 2"; do
  set -- $c
  python scripts/dense_one.py $1 $2 $3 > gpurun_out/dense_one_$1_$3.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dense_launch_$1_$3.csv python scripts/dense_one.py $1 $2 $3 > /dev/null 2>&1
done
ls gpurun_out
