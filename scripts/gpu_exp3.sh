set -x
mkdir -p gpurun_out
for f in 0 32 64 128; do
  timeout 300 scripts/sector_ubench 17 64,256,1024,16384 $f > gpurun_out/ubench_fetch$f.jsonl 2>> gpurun_out/ubench_fetch.err
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:k_independent -c 4 --csv scripts/sector_ubench 17 1024,16384 32 > gpurun_out/ncu_ubench32.csv 2>&1
bash scripts/exp_env.sh lj_full gpurun_out/exp_fetch_lj.jsonl "GEER_L2_FETCH=32" "GEER_L2_FETCH=64" "GEER_L2_FETCH=128" "GEER_L2_FETCH=0" "GEER_L2_FETCH=32 GEER_ARC_POLICY=2" > gpurun_out/exp_fetch.log 2>&1
