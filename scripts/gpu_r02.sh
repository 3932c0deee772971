#!/bin/bash
# Round-2 refresh on one GPU box (run from the repo root through gpurun):
#   tests   all `-m gpu` tests and smoke()
#   bench   the graded line (LJ-shaped config) and config 1
#   profile the ncu captures behind bench.py's roofline (K6 on the graded config, K9 q=16/64),
#           the per-batch walk-step counts, a launch list of the graded step
# Usage: bash scripts/gpu_r02.sh [tests|bench|profile|all]
set -x
PART=${1:-all}
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/build.log 2>&1
if [ "$PART" = tests ] || [ "$PART" = all ]; then
  timeout 3000 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1
  timeout 600 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
fi
if [ "$PART" = bench ] || [ "$PART" = all ]; then
  timeout 1200 python bench.py > gpurun_out/bench_lj.log 2>&1
  timeout 600 python bench.py --config rmat20 > gpurun_out/bench_rmat20.log 2>&1
fi
if [ "$PART" = profile ] || [ "$PART" = all ]; then
  CFG=lj_full
  timeout 600 python scripts/walk_batch_steps.py $CFG > gpurun_out/walk_steps_$CFG.json 2> gpurun_out/walk_steps_$CFG.err
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_walks -s 5 -c 1 -f \
      -o gpurun_out/walks_$CFG python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-spmm \
      --no-accuracy > gpurun_out/ncu_walks_$CFG.log 2>&1
  timeout 900 ncu --set full --clock-control none -k 'regex:k_spmm_(rows|items)' -s 3 -c 1 -f -o gpurun_out/spmm16_$CFG \
      python scripts/spmm_probe.py $CFG > gpurun_out/ncu_spmm16_$CFG.log 2>&1
  timeout 900 ncu --set full --clock-control none -k 'regex:k_spmm_(rows|items)' -s 11 -c 1 -f -o gpurun_out/spmm64_$CFG \
      python scripts/spmm_probe.py $CFG > gpurun_out/ncu_spmm64_$CFG.log 2>&1
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 800 --csv \
      --log-file gpurun_out/launches_$CFG.csv python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline \
      --no-spmm --no-accuracy > gpurun_out/ncu_launch_$CFG.log 2>&1
fi
ls -la gpurun_out | tail -30
if [ "$PART" = extra ]; then
  # the Orkut-shaped config; two real ranks on one GPU over gloo (plumbing); the Friendster-shaped
  # shard (configs[4], one GPU's 125k of 1M)
  timeout 900 python bench.py --config orkut_full --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_orkut.log 2>&1
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
      bench.py --gpus 2 --dist-backend gloo --config rmat20 --steps 3 --warmup 3 --no-cpu-baseline --no-spmm \
      --no-accuracy > gpurun_out/bench_2rank_gloo.log 2>&1
  timeout 1800 python bench.py --config friendster --steps 3 --warmup 3 --no-cpu-baseline --no-spmm > gpurun_out/bench_friendster.log 2>&1
  # the matching random-DRAM ceiling for K6 on the graded config (64-byte fetches, 256 MB - 1 GB buffers)
  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/sector_ubench scripts/sector_ubench.cu
  UBENCH_FLAVOURS=1 timeout 300 scripts/sector_ubench 2 128,256,512,1024 > gpurun_out/ubench_mid.jsonl 2>&1
  UBENCH_FLAVOURS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none \
      -k regex:k_flavour --csv scripts/sector_ubench 2 128,256,512,1024 > gpurun_out/ncu_ubench_mid.csv 2>&1
  # K6 on config 1 (packed layout): the capture behind its random_sector_l2 roofline
  timeout 600 python scripts/walk_batch_steps.py rmat20 > gpurun_out/walk_steps_rmat20.json 2> gpurun_out/walk_steps_rmat20.err
  timeout 900 ncu --set full --clock-control none -k regex:k_walks -s 5 -c 1 -f -o gpurun_out/walks_rmat20 \
      python bench.py --config rmat20 --steps 1 --warmup 1 --no-cpu-baseline --no-spmm --no-accuracy > gpurun_out/ncu_walks_rmat20.log 2>&1
fi
