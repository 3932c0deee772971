#!/bin/bash
# K6 ncu --set full capture + launch list on configs[3] (Orkut-shaped), so that its bench line
# carries the ncu-based K6 roofline like the graded config and config 1 (scripts/gpu_final.sh).
mkdir -p gpurun_out
CFG=orkut_full
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 800 --csv \
    --log-file gpurun_out/launches_$CFG.csv python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline \
    --no-spmm --no-accuracy > gpurun_out/ncu_launch_$CFG.log 2>&1
timeout 600 python scripts/walk_batch_steps.py $CFG > gpurun_out/walk_steps_$CFG.json 2> gpurun_out/walk_steps_$CFG.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_walks -s 5 -c 1 -f \
    -o gpurun_out/walks_$CFG python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-spmm \
    --no-accuracy > gpurun_out/ncu_walks_$CFG.log 2>&1
python scripts/ncu_summary.py walks gpurun_out/walks_$CFG.ncu-rep $CFG gpurun_out/walk_steps_$CFG.json \
    > gpurun_out/ncu_k_walks_${CFG}_final.json 2> gpurun_out/ncu_summary_$CFG.err
cat gpurun_out/ncu_k_walks_${CFG}_final.json | cut -c1-600
cp gpurun_out/ncu_k_walks_${CFG}_final.json profiles/ncu_k_walks_${CFG}_r02.json
timeout 900 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_orkut_ncu.log 2> gpurun_out/bench_orkut_ncu.err
tail -1 gpurun_out/bench_orkut_ncu.log | cut -c1-200
rm -f gpurun_out/walks_$CFG.ncu-rep.tmp
