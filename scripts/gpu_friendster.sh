# BASELINE config 4 (Friendster-shaped) on one B200: generation, graph creation, bench of one
# GPU's 125k-query shard of the 1M-query set
set -x
python __graft_entry__.py build > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/fr_mem.log
timeout 1200 python -c "
import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
import workloads as W
t = time.time(); g, pairs, _ = W.load_config('friendster')
print('gen', g.n, g.nnz, int(g.degrees().max()), round(time.time() - t, 1), 's', flush=True)
print('torch peak GB', torch.cuda.max_memory_allocated() / 1e9, flush=True)
import paper_2312_06123_b200 as G
t = time.time(); h = G.er_graph_create(g.n, g.offsets, g.cols); print('create', round(time.time() - t, 1), 's', flush=True)
t = time.time(); lam = G.er_graph_estimate_lambda(h); print('lambda', lam, round(time.time() - t, 1), 's', flush=True)
r, st = G.er_query_batch_ex(h, pairs[:2000], 0.1, stats=True)
print('2000 queries ok; mean steps', st['steps_total'].mean(), 'mean ell', st['ell'].mean(), flush=True)
" > gpurun_out/fr_gen.log 2>&1
cat gpurun_out/fr_gen.log
timeout 1500 python bench.py --config friendster --queries 125000 --steps 3 --warmup 3 --no-spmm --no-cpu-baseline > gpurun_out/bench_friendster.log 2>&1
tail -3 gpurun_out/bench_friendster.log | cut -c1-400
