mkdir -p gpurun_out
rm -f gpurun_out/abb_*.jsonl
for V in r0 r4 r5 r1; do
  GEER_LIB=$PWD/_varlib/$V.so timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_bkt_reduce_warp -c 12 --csv \
     --log-file gpurun_out/hab_$V.csv python bench.py --config lj_full --steps 1 --warmup 1 --no-cpu-baseline --no-spmm --no-accuracy > /dev/null 2>&1
done
bash scripts/ab_bench.sh lj_full 2 r0 r4 r5 r1
bash scripts/ab_bench.sh rmat20 2 r0 r4 r5 r1
cat gpurun_out/abb_*.jsonl
