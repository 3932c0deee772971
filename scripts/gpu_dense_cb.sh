set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
for cb in 8 16 32; do
  for c in "1000 0.05 2" "32 0.1 2"; do
    set -- $c
    GEER_HUB_CB=$cb python scripts/dense_one.py $1 $2 $3 > /dev/null 2>&1 && \
    GEER_HUB_CB=$cb ncu --metrics gpu__time_duration.sum --clock-control none -k regex:spmm --csv --log-file gpurun_out/cb${cb}_$1.csv python scripts/dense_one.py $1 $2 $3 > /dev/null 2>&1
  done
done
