#!/bin/bash
# K6 on configs[4] (Friendster-shaped, one GPU's 125k-query shard): launch list (single-pass time
# metric) and the DRAM / L2 counters of one K6 launch (batch 0 of the timed step).  Not --set full:
# the handle holds ~70 GB, so the capture is limited to the few counters the roofline needs.
mkdir -p gpurun_out
CFG=friendster
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 800 --csv \
    --log-file gpurun_out/launches_$CFG.csv python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline \
    --no-spmm --no-accuracy > gpurun_out/ncu_launch_$CFG.log 2>&1
echo "launch list rc=$?"
timeout 900 python scripts/walk_batch_steps.py $CFG > gpurun_out/walk_steps_$CFG.json 2> gpurun_out/walk_steps_$CFG.err
echo "walk steps rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors.sum
M=$M,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_ltcfabric.sum
M=$M,l1tex__m_xbar2l1tex_read_sectors_mem_lg_op_ld.sum,l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
M=$M,launch__registers_per_thread,launch__grid_size,dram__throughput.avg.pct_of_peak_sustained_elapsed
timeout 1500 ncu --metrics $M --clock-control none -k regex:k_walks -s 5 -c 1 -f \
    -o gpurun_out/walks_$CFG python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-spmm \
    --no-accuracy > gpurun_out/ncu_walks_$CFG.log 2>&1
echo "capture rc=$?"
python scripts/ncu_summary.py walks gpurun_out/walks_$CFG.ncu-rep $CFG gpurun_out/walk_steps_$CFG.json \
    > gpurun_out/ncu_k_walks_${CFG}_final.json 2> gpurun_out/ncu_summary_$CFG.err
cat gpurun_out/ncu_k_walks_${CFG}_final.json | cut -c1-1500
nvidia-smi --query-gpu=memory.used --format=csv,noheader
