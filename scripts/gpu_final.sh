#!/bin/bash
# Round-end refresh on one GPU box (everything the committed profiles/ and DESIGN.md cite):
#   tests + smoke; the graded bench line (LJ-shaped, full: cpu_baseline, K9, accuracy) and config 1;
#   K6 ncu --set full on both; launch lists of both; Orkut- and Friendster-shaped lines; the 2-rank
#   gloo plumbing run.
set -x
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1
timeout 600 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_lj.log 2>&1
timeout 600 python bench.py --config rmat20 > gpurun_out/bench_rmat20.log 2>&1
for CFG in lj_full rmat20; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 800 --csv \
      --log-file gpurun_out/launches_$CFG.csv python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline \
      --no-spmm --no-accuracy > gpurun_out/ncu_launch_$CFG.log 2>&1
  timeout 600 python scripts/walk_batch_steps.py $CFG > gpurun_out/walk_steps_$CFG.json 2> gpurun_out/walk_steps_$CFG.err
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_walks -s 5 -c 1 -f \
      -o gpurun_out/walks_$CFG python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-spmm \
      --no-accuracy > gpurun_out/ncu_walks_$CFG.log 2>&1
  python scripts/ncu_summary.py walks gpurun_out/walks_$CFG.ncu-rep $CFG gpurun_out/walk_steps_$CFG.json \
      > gpurun_out/ncu_k_walks_${CFG}_final.json 2> gpurun_out/ncu_summary_$CFG.err
done
timeout 900 ncu --set full --clock-control none -k 'regex:k_spmm_(rows|items)' -s 3 -c 1 -f -o gpurun_out/spmm16_rmat20 \
    python scripts/spmm_probe.py rmat20 > gpurun_out/ncu_spmm16_rmat20.log 2>&1
timeout 900 ncu --set full --clock-control none -k 'regex:k_spmm_(rows|items)' -s 11 -c 1 -f -o gpurun_out/spmm64_rmat20 \
    python scripts/spmm_probe.py rmat20 > gpurun_out/ncu_spmm64_rmat20.log 2>&1
python scripts/ncu_summary.py spmm gpurun_out/spmm16_rmat20.ncu-rep rmat20 16 > gpurun_out/ncu_k_spmm_q16_rmat20.json 2>/dev/null
python scripts/ncu_summary.py spmm gpurun_out/spmm64_rmat20.ncu-rep rmat20 64 > gpurun_out/ncu_k_spmm_q64_rmat20.json 2>/dev/null
timeout 900 python bench.py --config orkut_full --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_orkut.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --dist-backend gloo --config rmat20 --steps 3 --warmup 3 --no-cpu-baseline --no-spmm \
    --no-accuracy > gpurun_out/bench_2rank_gloo.log 2>&1
timeout 2400 python bench.py --config friendster --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_friendster.log 2>&1
ls -la gpurun_out | tail -40
